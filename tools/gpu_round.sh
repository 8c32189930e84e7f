# Round check on one GPU: build, smoke, the GPU test suite, the default bench
# line.  bash tools/gpu_round.sh [out_dir]
O=${1:-gpurun_out/round}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 400 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
python -c "import json;d=json.loads(open(\"$O/bench.json\").read().strip().splitlines()[-1]);print({k:d.get(k) for k in (\"value\",\"p50_ms\",\"p99_ms\",\"l2_stretch\",\"gpu_launches\")});print(d[\"roofline\"]);print(d.get(\"latency_floor\"))"
