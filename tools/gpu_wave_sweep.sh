# p50 pack time vs wave size (TABI_WAVE) on C3 / C2 / C4
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for W in ${WORKLOADS:-C3 C2}; do
for B in ${WAVES:-1 2 4 8 16}; do
  TABI_WAVE=$B timeout 300 python bench.py --workload $W --steps 100 --warmup 5 > gpurun_out/sweep_${W}_$B.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/sweep_${W}_$B.json')); print('$W', 'B=$B', round(d['ms_per_step']*1000,1), 'us  p99', round(d['p99_ms']*1000,1))"
done; done
