mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python tools/profile_once.py --workload C4 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 24 -c 8 --csv --log-file gpurun_out/launches_C4.csv python tools/profile_once.py --workload C4 > gpurun_out/ncu_list.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pack_kernel|proxy_kernel|sort_kernel" -s 3 -c 3 -o gpurun_out/prof_c4 python tools/profile_once.py --workload C4 > gpurun_out/ncu_c4.log 2>&1
echo "rc=$?"
