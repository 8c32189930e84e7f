# ncu --set full of one kernel (regex $1) of the 4th pack
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
K=${1:-profile_kernel}
python tools/profile_once.py > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$K" -s 3 -c 1 -o gpurun_out/prof_$K python tools/profile_once.py > gpurun_out/ncu_$K.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_$K.log
