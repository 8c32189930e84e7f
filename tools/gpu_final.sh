# Round-end evidence: bench lines (default C5 batch line + every single-pack
# workload + the reference arm), ncu launch lists and --set full captures of
# the dominant kernels (C3 / C4: fused + proxy; C5: many + proxy).
#   bash tools/gpu_final.sh [out]
O=${1:-gpurun_out/final}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
lscpu > $O/lscpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?"
for W in C3 C2 C4 C4P C4X; do
  timeout 600 python bench.py --workload $W > $O/bench_$W.json 2> $O/bench_$W.err; echo "bench $W rc=$?"
done
timeout 600 python bench.py --workload C3 --rho 2.0 > $O/bench_rho2.json 2>/dev/null; echo "rho2 rc=$?"
timeout 600 python bench.py --workload C3 --rho 0.5 > $O/bench_rho05.json 2>/dev/null; echo "rho0.5 rc=$?"
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference.json 2>/dev/null; echo "ref rc=$?"
for W in C3 C4 C5; do
  python tools/profile_once.py --workload $W > $O/plain_$W.log 2>&1 || { echo "plain $W failed"; continue; }
  L=$(grep -o 'launches/pack [0-9]*' $O/plain_$W.log | awk '{print $2}')
  ncu --metrics gpu__time_duration.sum --clock-control none -s $((3*L)) -c $L --csv \
      --log-file $O/launches_$W.csv python tools/profile_once.py --workload $W > $O/ncu_list_$W.log 2>&1
  echo "list $W rc=$?"
  KS="fused_kernel proxy_kernel"; [ $W = C5 ] && KS="many_kernel proxy_kernel"
  for K in $KS; do
    ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
        -o $O/prof_${K}_$W python tools/profile_once.py --workload $W > $O/ncu_${K}_$W.log 2>&1
    echo "$K $W rc=$?"
  done
done
