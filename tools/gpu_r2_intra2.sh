#!/bin/bash
# k_intra_tw split by segment length: parity of the VRPTW intra paths + kernel times (two register budgets)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 1200 python -m pytest tests -q -m gpu -x -k "vrptw or intra or tw or fields or reversed or pd" 2>&1 | tail -3
for v in lb3 lb1; do
  if [ $v = lb1 ]; then
    sed -i 's/__launch_bounds__(256, 3) k_intra_tw/__launch_bounds__(256) k_intra_tw/' paper_2506_17357_b200/csrc/tga_kernels.cu
    python paper_2506_17357_b200/build.py --force > /dev/null 2>&1
  fi
  for c in cfg3r2 cfg3; do
    timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_intra|k_inter" -c 12 --csv \
      python tools/prof_eval.py --config $c --mask all --reps 6 2>/dev/null | grep -E "k_intra|k_inter" | \
      python -c "
import sys,csv,collections
d=collections.defaultdict(list)
for r in csv.reader(sys.stdin):
    if len(r)>10 and r[-3]=='gpu__time_duration.sum': d[r[4].split('(')[0][:40]].append(float(r[-1]))
for k,v in d.items(): print('$v $c', k, 'n', len(v), 'median %.2f' % sorted(v)[len(v)//2], r[-2] if False else '')
"
  done
  timeout 600 python bench.py --config cfg3r2 --no-cpu-baseline --no-per-op --no-north-star --no-row-shard --steps 60 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v cfg3r2 us/step %.2f marginal %s' % (1e3*d['ms_per_step'], d.get('us_per_step_marginal')))"
done
