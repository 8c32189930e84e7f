# one GPU call: tests, bench, launch list
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/bench.err
for W in C2 C4 C4P; do timeout 300 python bench.py --steps 10 --warmup 3 --workload $W --no-cpu-baseline > gpurun_out/bench_$W.json 2>&1; done
timeout 300 python bench.py --steps 20 --warmup 3 --rho 2.0 --no-cpu-baseline > gpurun_out/bench_rho2.json 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --workload C5 --no-cpu-baseline > gpurun_out/bench_C5.json 2>&1; echo "c5 rc=$?"
