#!/bin/bash
# compute-sanitizer over every kernel entry point (memcheck, racecheck, synccheck, initcheck)
# on cfg1 / cfg2 / small VRPTW / a small batch, both score modes.  Summaries -> gpurun_out/sanitize_*.txt
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for tool in memcheck racecheck synccheck initcheck; do
  for w in cfg1 vrptw pd batch cfg2 ns2000; do
    [ "$tool" = racecheck ] && { [ "$w" = cfg2 ] || [ "$w" = ns2000 ]; } && continue   # racecheck at n >= 1000: too slow, cfg1 covers the same code
    timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_driver.py $w \
      > gpurun_out/sanitize_${tool}_${w}.txt 2>&1
    echo "$tool $w rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_${tool}_${w}.txt | tail -1)"
  done
done
