# Round profile: per-kernel launch list (ncu gpu__time_duration, one pack) and
# --set full captures of the fused wave kernel and the proxy kernel.
#   bash tools/gpu_profile_round.sh [C3|C4|C2]
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
W=${1:-C3}
python tools/profile_once.py --workload $W > gpurun_out/plain_$W.log 2>&1 || { echo "plain run failed"; exit 1; }
L=$(grep -o 'launches/pack [0-9]*' gpurun_out/plain_$W.log | awk '{print $2}')
echo "launches/pack $L"
ncu --metrics gpu__time_duration.sum --clock-control none -s $((3*L)) -c $L --csv \
    --log-file gpurun_out/launches_$W.csv python tools/profile_once.py --workload $W > gpurun_out/ncu_list_$W.log 2>&1
echo "list rc=$?"
for K in fused_kernel proxy_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
      -o gpurun_out/prof_${K}_$W python tools/profile_once.py --workload $W > gpurun_out/ncu_${K}_$W.log 2>&1
  echo "$K rc=$?"
done
