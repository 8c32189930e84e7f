# fused-kernel trace for raster group counts 1, 2, 4 (stage + timeline only)
mkdir -p gpurun_out
for RG in 1 2 4; do
  TABI_NVCC_EXTRA="-DTABI_FUSED_RG=$RG" python -c "from paper_2602_07782_b200 import build as b; b.build(force=True)" > gpurun_out/build_rg$RG.log 2>&1
  echo "=== RG=$RG"
  TRACE_MODES=1 timeout 300 python tools/fused_trace.py 2>&1 | sed 's/rows.*//'
done
