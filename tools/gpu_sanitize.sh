# compute-sanitizer memcheck on one small pack (fused and split paths)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for F in 0 1; do
  echo "== TABI_FUSED=$F"
  TABI_FUSED=$F timeout 600 compute-sanitizer --tool memcheck --show-backtrace no --print-limit 5 python tools/profile_once.py --workload ${W:-C2} --warmup 0 2>&1 | grep -v "^=========     " | head -40
done
