#!/bin/bash
# K-dependence of the bench line (ms_per_step vs marginal) + warp-TW intra on R1
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for c in cfg3r2 cfg2; do for K in 20 60 180; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-per-op --no-north-star --no-row-shard --steps $K 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c K=$K us/step %.2f marginal %s fixed %s applied %s reps %s' % (1e3*d['ms_per_step'], d.get('us_per_step_marginal'), d.get('graph_launch_fixed_us'), d.get('applied_moves'), d['config'].get('l2')))"
done; done
for w in 0 1; do
  TGA_WARP_TW=$w timeout 600 python bench.py --config cfg3 --no-cpu-baseline --no-per-op --no-north-star --no-row-shard --steps 60 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg3 warp_tw=$w us/step %.2f marginal %s' % (1e3*d['ms_per_step'], d.get('us_per_step_marginal')))"
done
