# source-level stall sampling of the split-path packer alone (C3, one candidate),
# densest sampling interval
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
export TABI_FUSED=0 TABI_WAVE=1
python tools/profile_once.py --workload C3 > gpurun_out/plain.log 2>&1 || { echo "plain failed"; exit 1; }
ncu --section SourceCounters --section WarpStateStats --warp-sampling-interval 0 --clock-control none --import-source on -k regex:pack_kernel -s 3 -c 1 \
   -o gpurun_out/prof_pack_dense_C3 python tools/profile_once.py --workload C3 > gpurun_out/ncu_pk2.log 2>&1; echo "pack rc=$?"
