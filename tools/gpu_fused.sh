# one GPU call: fused-kernel parity + bench (fused vs split)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 --timeout-method thread > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for F in 1 0; do
  TABI_FUSED=$F timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_C3_f$F.json 2>&1; echo "c3 f$F rc=$?"
  TABI_FUSED=$F timeout 300 python bench.py --steps 10 --warmup 3 --workload C4 --no-cpu-baseline > gpurun_out/bench_C4_f$F.json 2>&1; echo "c4 f$F rc=$?"
  TABI_FUSED=$F timeout 300 python bench.py --steps 10 --warmup 3 --workload C2 --no-cpu-baseline > gpurun_out/bench_C2_f$F.json 2>&1
done
