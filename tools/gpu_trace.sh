# K4 row-phase trace (a -DTABI_PHASE_TRACE build) of the winner's chain alone
# (one candidate per wave) and with the default waves.
#   bash tools/gpu_trace.sh [sets] [out]      sets: comma list of C3,C3r15,C2,C4
S=${1:-C3r15,C3}
O=${2:-gpurun_out/trace}
mkdir -p $O
TABI_NVCC_EXTRA=-DTABI_PHASE_TRACE python -c "from paper_2602_07782_b200 import build as b; b.build(force=True)" > $O/build_trace.log 2>&1
echo "== TABI_WAVE=1"
TABI_WAVE=1 TRACE_SETS=$S TRACE_MODES=1 timeout 300 python tools/fused_trace.py 2>&1 | tee $O/trace_wave1.txt
echo "== default waves"
TRACE_SETS=$S TRACE_MODES=1 timeout 300 python tools/fused_trace.py 2>&1 | tee $O/trace_default.txt
python -c "from paper_2602_07782_b200 import build as b; b.build(force=True)" > $O/build.log 2>&1
