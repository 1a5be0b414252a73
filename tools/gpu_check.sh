#!/bin/bash
# One GPU session: parity tests, bench lines, launch list, one full ncu capture of the top kernel.
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
timeout 600 python bench.py --config ns2000 --no-cpu-baseline > gpurun_out/bench_ns2000.json 2> gpurun_out/bench_ns2000.err
timeout 600 python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu-baseline --no-per-op > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 600 python bench.py --config cfg5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python tools/prof_dev.py --config cfg2 --steps 6 > gpurun_out/launches_cfg2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_inter_fast -s 4 -c 1 -o gpurun_out/prof_fast_ns2000 python tools/prof_dev.py --config ns2000 --steps 6 > gpurun_out/prof_ns2000.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_inter_fast -s 4 -c 1 -o gpurun_out/prof_fast_cfg2 python tools/prof_dev.py --config cfg2 --steps 6 > gpurun_out/prof_cfg2.log 2>&1
ls -la gpurun_out
