"""The cross-GPU combine (BASELINE.json north_star "partial
best moves combined with an NCCL allreduce ... packed as (delta, index) so the
combine is exact") executed for real on one GPU: a world-1 NCCL communicator
created through the C ABI (tga_nccl_unique_id / tga_comm_init), so every tga_eval
ends with ncclAllReduce(MIN, uint64) on the solution's stream.  With one rank the
allreduce is the identity, so the keys must equal the unsharded evaluation's --
eagerly, inside a captured CUDA graph, and through device-resident steps.
(Several ranks need several GPUs; their host logic is tests/test_dist_gloo.py.)"""
import numpy as np
import pytest

import tga_gen as G
from tests.conftest import gpu_available

pytestmark = pytest.mark.gpu

if gpu_available():
    import torch
    from paper_2506_17357_b200 import tga as T
else:  # pragma: no cover
    T = None


def _need_gpu():
    if not gpu_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("name", ["cvrp", "vrptw"])
def test_world1_communicator_keys_equal_unsharded(name):
    _need_gpu()
    if name == "cvrp":
        inst, sol = G.x_like(4, n=400, target_routes=17)
        masks = [T.OP_ALL, T.OP_FUSED_NS, T.OP_INTER]
    else:
        inst, sol = G.gh_like(4, n=300, kind="R1")
        masks = [T.OP_ALL & ~T.OP_2OPT, T.OP_INTER]
    gi = T.Instance.from_gen(inst)
    ref = T.Solution(gi, sol)
    com = T.Solution(gi, sol)
    com.comm_init(0, 1, T.nccl_unique_id())
    for m in masks:
        ref.eval(m)
        com.eval(m)
        np.testing.assert_array_equal(com.keys(), ref.keys())


def test_world1_communicator_in_graph_and_device_steps():
    """Evals with the allreduce captured in a CUDA graph and replayed; then 25
    device-resident steps (eval + allreduce + on-device pick / apply) follow the
    trajectory of a solution without a communicator."""
    _need_gpu()
    inst, sol = G.x_like(5, n=300, target_routes=13)
    gi = T.Instance.from_gen(inst)
    ref = T.Solution(gi, sol)
    com = T.Solution(gi, sol)
    com.comm_init(0, 1, T.nccl_unique_id())
    st = torch.cuda.Stream()
    com.set_stream(st)
    com.eval(T.OP_ALL, st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(4):
            com.eval(T.OP_ALL, st)
    g.replay()
    torch.cuda.synchronize()
    ref.eval(T.OP_ALL)
    np.testing.assert_array_equal(com.keys(), ref.keys())
    for _ in range(25):
        ref.step_async(T.OP_ALL)
        com.step_async(T.OP_ALL)
    assert com.routes() == ref.routes()
    assert com.device_stats()[1] == ref.device_stats()[1]
