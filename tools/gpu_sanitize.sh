# compute-sanitizer evidence on one small pack: memcheck, racecheck (shared
# memory hazards) and synccheck (barrier misuse), fused and split paths.
#   W=C2 bash tools/gpu_sanitize.sh     -> gpurun_out/sanitize/<tool>_<path>.txt
mkdir -p gpurun_out/sanitize
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
W=${W:-C2}
for F in 1 0; do
  P=$([ $F = 1 ] && echo fused || echo split)
  for T in memcheck racecheck synccheck; do
    EXTRA=""
    [ $T = racecheck ] && EXTRA="--racecheck-report all"
    TABI_FUSED=$F timeout 1200 compute-sanitizer --tool $T $EXTRA --show-backtrace no --print-limit 20 \
      python tools/profile_once.py --workload $W --warmup 0 > gpurun_out/sanitize/${T}_${P}_$W.txt 2>&1
    echo "$T $P rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/sanitize/${T}_${P}_$W.txt | tail -2 | tr '\n' ' ')"
  done
done
