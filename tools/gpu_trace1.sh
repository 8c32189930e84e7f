# fused-kernel trace (phase-trace build); env passes through (e.g. TABI_WAVE)
mkdir -p gpurun_out
TABI_NVCC_EXTRA=-DTABI_PHASE_TRACE python -c "from paper_2602_07782_b200 import build as b; b.build(force=True)" > gpurun_out/build_trace.log 2>&1
for B in ${WAVES:-16}; do
echo "== TABI_WAVE=$B"
TABI_WAVE=$B TRACE_MODES=1 timeout 300 python tools/fused_trace.py 2>&1 | head -${NLINES:-3}
done
