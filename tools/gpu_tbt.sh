# one GPU call: parity tests, default bench, then the phase trace (B=1 and default)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 --timeout-method thread > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for W in ${WORKLOADS:-C3}; do
timeout 300 python bench.py --workload $W > gpurun_out/bench_$W.json 2> gpurun_out/bench.err; echo "bench $W rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_$W.json')); print('$W', d['value'], d['ms_per_step'], d['e2e']['value'])"
done
if [ -n "$TRACE" ]; then WAVES="${TRACE}" NLINES=${NLINES:-1} bash tools/gpu_trace1.sh; fi
