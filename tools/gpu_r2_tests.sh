#!/bin/bash
# GPU parity suite (+ optional -k filter via PYTEST_K) and smoke
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1 || { tail -20 gpurun_out/smoke.log; exit 1; }
timeout 2400 python -m pytest tests -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} --durations=15 > gpurun_out/pytest_gpu.log 2>&1
tail -30 gpurun_out/pytest_gpu.log
