# one GPU call: tests, bench, launch list
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 300 python bench.py --steps 20 --warmup 3 --workload C2 --no-cpu-baseline > gpurun_out/bench_c2.json 2>&1; cat gpurun_out/bench_c2.json | tail -2
timeout 300 python bench.py --steps 20 --warmup 3 --rho 2.0 --no-cpu-baseline > gpurun_out/bench_rho2.json 2>&1; tail -2 gpurun_out/bench_rho2.json
