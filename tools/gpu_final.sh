# Round-end evidence: bench lines (all workloads + reference arm), launch lists
# and --set full captures (fused + proxy kernels) for C3 and C4.
mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/final/build.log 2>&1
for W in C3 C2 C4 C4P C4X; do
  timeout 600 python bench.py --workload $W > gpurun_out/final/bench_$W.json 2> gpurun_out/final/bench_$W.err; echo "bench $W rc=$?"
done
timeout 600 python bench.py --workload C3 --rho 2.0 > gpurun_out/final/bench_rho2.json 2>/dev/null; echo "rho2 rc=$?"
timeout 900 python bench.py --impl reference --steps 30 --warmup 3 > gpurun_out/final/bench_reference.json 2>/dev/null; echo "ref rc=$?"
for W in C3 C4; do
  python tools/profile_once.py --workload $W > gpurun_out/final/plain_$W.log 2>&1 || { echo "plain $W failed"; continue; }
  L=$(grep -o 'launches/pack [0-9]*' gpurun_out/final/plain_$W.log | awk '{print $2}')
  ncu --metrics gpu__time_duration.sum --clock-control none -s $((3*L)) -c $L --csv \
      --log-file gpurun_out/final/launches_$W.csv python tools/profile_once.py --workload $W > gpurun_out/final/ncu_list_$W.log 2>&1
  echo "list $W rc=$?"
  for K in fused_kernel proxy_kernel; do
    ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
        -o gpurun_out/final/prof_${K}_$W python tools/profile_once.py --workload $W > gpurun_out/final/ncu_${K}_$W.log 2>&1
    echo "$K $W rc=$?"
  done
done
