# bench C3 under the three flush modes (diagnostic)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for F in write write+read none; do
  timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --flush $F > gpurun_out/bench_flush_$F.json 2>&1; echo "$F rc=$?"
done
