# one GPU call: parity tests (normal build), then the fused trace (phase-trace build)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 --timeout-method thread > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/fused_trace.py 2>&1 | sed 's/ns\/row.*//'
TABI_NVCC_EXTRA=-DTABI_PHASE_TRACE python -c "from paper_2602_07782_b200 import build as b; b.build(force=True)" > gpurun_out/build_trace.log 2>&1
TRACE_MODES=1 timeout 300 python tools/fused_trace.py 2>&1 | sed 's/.*rows/rows/'
