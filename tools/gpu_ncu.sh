# ncu: launch list (all kernels of the 4th pack) + one --set full capture of the top kernels
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python tools/profile_once.py > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 24 -c 8 --csv --log-file gpurun_out/launches.csv python tools/profile_once.py > gpurun_out/ncu_list.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"profile_kernel|pack_kernel|proxy_kernel" -s 9 -c 3 -o gpurun_out/prof python tools/profile_once.py > gpurun_out/ncu_full.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/ncu_full.log
cat gpurun_out/launches.csv | tail -12
