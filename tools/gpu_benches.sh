#!/bin/bash
# Every bench line of profiles/: default (cfg2 + CPU oracle), the other configs, the reference arm.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/b_cfg2.json 2> gpurun_out/b_cfg2.err
for c in ns2000 cfg3 cfg3r2; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err; done
timeout 600 python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu-baseline --no-per-op > gpurun_out/b_cfg4.json 2> gpurun_out/b_cfg4.err
timeout 600 python bench.py --config cfg5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/b_cfg5.json 2> gpurun_out/b_cfg5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/b_reference.json 2> gpurun_out/b_reference.err
for f in gpurun_out/b_*.json; do echo "$f $(head -c 300 $f)"; done
