#!/bin/bash
# bench lines: penalised vs feasible cfg2, cfg5 population, into gpurun_out/
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for spec in "cfg2 feasible" "cfg2 penalised" "cfg4 penalised" "cfg5 feasible"; do
  set -- $spec
  timeout 900 python bench.py --config $1 --score $2 --no-cpu-baseline --no-north-star --no-row-shard > gpurun_out/line_$1_$2.json 2> gpurun_out/line_$1_$2.err
  python -c "import json; d=json.loads(open('gpurun_out/line_$1_$2.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$1 $2 us/step %.2f value %.3g kernel %.2f us frac %.3f traffic %s' % (1e3*d['ms_per_step'], d['value'], 1e3*r['kernel_ms'], r['frac'], r.get('traffic')))"
done
