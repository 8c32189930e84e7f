# per-kernel device times of the 4th pack (ncu launch list, cold-cache/serialised)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
W=${1:-C3}
python tools/profile_once.py --workload $W > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 24 -c 8 --csv --log-file gpurun_out/launches_$W.csv python tools/profile_once.py --workload $W > gpurun_out/ncu_list.log 2>&1
echo "rc=$?"
python - <<'PY'
import csv, sys
rows = list(csv.reader(open(f"gpurun_out/launches_{sys.argv[1] if len(sys.argv)>1 else 'C3'}.csv")))
PY
