# --set full capture of the split-path pack_kernel on C3 with one candidate
# (TABI_FUSED=0 TABI_WAVE=1): every sample is the packer's row chain
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
export TABI_FUSED=0 TABI_WAVE=1
python tools/profile_once.py --workload C3 > gpurun_out/plain.log 2>&1 || { echo "plain failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:pack_kernel -s 3 -c 1 \
   -o gpurun_out/prof_pack_w1_C3 python tools/profile_once.py --workload C3 > gpurun_out/ncu_pk.log 2>&1; echo "pack rc=$?"
