# raster tile size sweep (fused kernel timeline)
for TC in 2048 4096 8192; do
  TABI_NVCC_EXTRA="-DTABI_TILE_CELLS=$TC" python -c "from paper_2602_07782_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  echo "== TILE_CELLS $TC"
  TRACE_MODES=1 timeout 300 python tools/fused_trace.py 2>&1 | sed 's/rows.*//'
done
