#!/bin/bash
# shared-staged route rebuild in the pick kernel + split VRPTW intra: parity, phases, step times
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for st in 1 0; do
  export TGA_SCAN_STAGE=$st
  for c in cfg2 cfg3r2 cfg4; do python tools/probe_step.py --config $c --steps 8 2>&1 | tail -1 | sed "s/^/stage=$st $c /"; done
  for c in cfg2 cfg3r2 cfg3; do python tools/step_times.py --config $c --steps 200 | sed "s/^/stage=$st /" | cut -c1-140; done
done
unset TGA_SCAN_STAGE
bash tools/gpu_r2_smi.sh
