mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/profile_once.py --workload C4 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:prep_kernel -s 1 -c 1 -o gpurun_out/prof_prep_C4 python tools/profile_once.py --workload C4 > gpurun_out/ncu_prep.log 2>&1; echo rc=$?
