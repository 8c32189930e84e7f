# --set full capture of the fused kernel on C3 with one candidate per wave
# (TABI_WAVE=1: the packer's row chain alone), plus the proxy kernel
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TABI_WAVE=1 python tools/profile_once.py --workload C3 > gpurun_out/plain.log 2>&1 || { echo "plain failed"; exit 1; }
TABI_WAVE=1 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 3 -c 1 \
   -o gpurun_out/prof_fused_w1_C3 python tools/profile_once.py --workload C3 > gpurun_out/ncu_f.log 2>&1; echo "fused rc=$?"
ncu --set full --clock-control none --import-source on -k regex:proxy_kernel -s 3 -c 1 \
   -o gpurun_out/prof_proxy_C3 python tools/profile_once.py --workload C3 > gpurun_out/ncu_p.log 2>&1; echo "proxy rc=$?"
