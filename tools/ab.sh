#!/bin/bash
# A/B step times of prebuilt libraries on one box: every tools/ab/libtga_*.so and the in-tree libtga.so
# usage (on the box): bash tools/ab.sh [configs...]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
CFGS=${@:-cfg2}
for rep in 1 2 3; do
  for L in tools/ab/libtga_*.so paper_2506_17357_b200/libtga.so; do
    tag=$(basename $L .so)
    for c in $CFGS; do
      TGA_LIB=$PWD/$L timeout 600 python bench.py --config $c --no-cpu-baseline --no-per-op --no-north-star --no-row-shard 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%-12s $c us/step %.2f marginal %.2f kernel %.2f' % ('$tag', 1e3*d['ms_per_step'], d.get('us_per_step_marginal') or -1, 1e3*d['roofline']['kernel_ms']))"
    done
  done
done
