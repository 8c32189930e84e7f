# A/B of a compile-time switch with the phase trace: bash tools/gpu_ab.sh "-DFLAG"
for X in "" "$1"; do
  TABI_NVCC_EXTRA="-DTABI_PHASE_TRACE $X" python -c "from paper_2602_07782_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  echo "== extra: '$X'"
  TRACE_MODES=${TRACE_MODES:-1,0} timeout 300 python tools/fused_trace.py 2>&1 | sed 's/raster ns.*//' | sed 's/stages_us.*rows/rows/'
done
