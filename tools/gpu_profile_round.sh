# Round profile of one workload: plain run, then the ncu launch list (device
# time of every kernel of one call) and --set full captures of the given
# kernels.   bash tools/gpu_profile_round.sh C5 "proxy_kernel many_kernel" [out_dir]
W=${1:-C5}
KS=${2:-"proxy_kernel many_kernel"}
O=${3:-gpurun_out/prof}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python tools/profile_once.py --workload $W > $O/plain_$W.log 2>&1 || { echo "plain run failed"; cat $O/plain_$W.log; exit 1; }
L=$(grep -o 'launches/pack [0-9]*' $O/plain_$W.log | awk '{print $2}')
echo "launches/pack $L"
ncu --metrics gpu__time_duration.sum --clock-control none -s $((3*L)) -c $L --csv \
    --log-file $O/launches_$W.csv python tools/profile_once.py --workload $W > $O/ncu_list_$W.log 2>&1
echo "list rc=$?"
for K in $KS; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 \
      -o $O/prof_${K}_$W python tools/profile_once.py --workload $W > $O/ncu_${K}_$W.log 2>&1
  echo "$K rc=$?"
done
