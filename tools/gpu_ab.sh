# A/B of compile-time variants on the latency and batch workloads.
#   bash tools/gpu_ab.sh "-DTABI_FUSED_RG=2" "-DTABI_FUSED_RG=4" ...
# (the empty variant -- the default build -- always runs first; the default
# build is restored at the end)
O=${AB_OUT:-gpurun_out/ab}
mkdir -p $O
for V in "" "$@"; do
  TABI_NVCC_EXTRA="$V" python -c "from paper_2602_07782_b200 import build as b; b.build(force=True)" > $O/build.log 2>&1 || { echo "build failed: $V"; tail -5 $O/build.log; continue; }
  echo "=== variant '$V'"
  timeout 300 python tools/c3_seeds.py --rho 1.5 | tail -9
  for R in 0.5; do
    timeout 300 python bench.py --workload C3 --rho $R --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C3 rho', $R, 'p50', round(d['p50_ms'],4), 'p99', round(d['p99_ms'],4), {k: round(v, 4) for k, v in d['stage_ms'].items()})"
  done
  for W in C2 C4; do
    timeout 300 python bench.py --workload $W --steps 30 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$W p50', round(d['p50_ms'],4), 'p99', round(d['p99_ms'],4))"
  done
  [ -z "$AB_NO_BATCH" ] && timeout 300 python tools/many_probe.py --reps 2
done
python -c "from paper_2602_07782_b200 import build as b; b.build(force=True)" > $O/build.log 2>&1
