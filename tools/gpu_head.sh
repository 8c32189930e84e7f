for H in 0 16384 65536; do
  TABI_NVCC_EXTRA="-DTABI_HEAD_CELLS=$H" python -c "from paper_2602_07782_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  echo "== HEAD $H"
  TRACE_MODES=1 timeout 300 python tools/fused_trace.py 2>&1 | sed 's/rows.*//'
done
