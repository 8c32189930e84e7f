# A/B of compile-time flags: phase trace (TABI_WAVE=1 and default) + p50 bench per variant
#   VARIANTS="'' '-DX=1'" bash tools/gpu_ab2.sh
mkdir -p gpurun_out
eval "set -- $VARIANTS"
for X in "$@"; do
  echo "=== extra: '$X'"
  TABI_NVCC_EXTRA="-DTABI_PHASE_TRACE $X" python -c "from paper_2602_07782_b200 import build as b; b.build(force=True)" > gpurun_out/build_ab.log 2>&1 || { echo build failed; tail -5 gpurun_out/build_ab.log; continue; }
  for B in ${WAVES:-1}; do
    TABI_WAVE=$B TRACE_MODES=1 timeout 300 python tools/fused_trace.py 2>&1 | head -${NLINES:-1} | sed 's/raster ns.*//'
  done
  TABI_NVCC_EXTRA="$X" python -c "from paper_2602_07782_b200 import build as b; b.build(force=True)" > gpurun_out/build_ab.log 2>&1
  for W in ${WORKLOADS:-C3}; do
    timeout 300 python bench.py --workload $W --steps 100 > gpurun_out/ab.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$W p50 us', round(d['ms_per_step']*1000,1))"
  done
done
