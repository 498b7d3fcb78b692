"""Data-parallel training host logic on CPU: world_size 2 over gloo.

paper_2406_00809_b200.dp drives an oracle-backed engine here: the reference
restatement's batch loss/gradient (oracle batch_loss_grads) and its Adam
(oracle adam_step). On the GPU box the same driver runs the C-ABI trainer over
NCCL. Two ranks, each on half the columns, must reproduce the single-process
full-batch training trajectory (gradient all-reduce = the reference's column
accumulate, src/gnn.cpp:439-440)."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from paper_2406_00809_b200.dp import DataParallelTrainer, shard_columns  # noqa: E402

DIMS = (4, 8, 2)
GLOBAL_B = 4
STEPS = 3
LR = 1e-2


class OracleEngine:
    def __init__(self, oc, a, params):
        import torch

        self.oc, self.a = oc, a
        self.p = np.array(params, np.float64)
        self.m1 = np.zeros_like(self.p)
        self.m2 = np.zeros_like(self.p)
        self.t = 0
        self.g = torch.zeros(len(self.p), dtype=torch.float64)

    def backward(self, x, b):
        k = x.shape[1]
        loss, grads = self.oc.batch_loss_grads(self.a, DIMS, self.p, np.asfortranarray(x).ravel(order="F"),
                                               np.asfortranarray(b).ravel(order="F"), k)
        self.g.copy_(__import__("torch").from_numpy(grads))
        return loss

    def backward_synthetic(self, seed):
        raise NotImplementedError

    def grad_tensor(self):
        return self.g

    def apply_grads(self):
        self.p, self.m1, self.m2, self.t = self.oc.adam_step(DIMS, self.p, self.g.numpy(), self.m1, self.m2,
                                                             self.t, LR)


def problem():
    import oracle

    oc = oracle.restatement()
    a = oc.prescale(oc.gen_convection_diffusion(6, 0.3), 8.6)
    params = oc.init_params(*DIMS, 0)
    xs, bs = [], []
    for s in range(STEPS):
        x, b = oc.gaussian_batch(a, 5, s, GLOBAL_B)
        xs.append(x.reshape(GLOBAL_B, a.n).T.copy())
        bs.append(b.reshape(GLOBAL_B, a.n).T.copy())
    return oc, a, params, xs, bs


def _worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        oc, a, params, xs, bs = problem()
        dp = DataParallelTrainer(OracleEngine(oc, a, params))
        losses = [dp.step(xs[s], bs[s]) for s in range(STEPS)]
        np.savez(f"{out}_{rank}.npz", params=dp.e.p, losses=np.array(losses), m1=dp.e.m1)
    finally:
        dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_columns():
    assert shard_columns(8, 0, 2) == slice(0, 4)
    assert shard_columns(8, 1, 2) == slice(4, 8)
    assert shard_columns(32, 3, 4) == slice(24, 32)
    with pytest.raises(ValueError):
        shard_columns(6, 0, 4)
    with pytest.raises(ValueError):
        shard_columns(8, 2, 2)


def test_dp_world2_matches_single_process(tmp_path):
    import torch.multiprocessing as mp

    out = str(tmp_path / "dp")
    mp.start_processes(_worker, args=(2, free_port(), out), nprocs=2, join=True, start_method="spawn")
    r0, r1 = np.load(f"{out}_0.npz"), np.load(f"{out}_1.npz")
    # replicas stay bit-identical
    assert np.array_equal(r0["params"], r1["params"])
    assert np.array_equal(r0["losses"], r1["losses"])
    # and follow the single-process full-batch trajectory
    oc, a, params, xs, bs = problem()
    ref = OracleEngine(oc, a, params)
    ref_losses = []
    for s in range(STEPS):
        ref_losses.append(ref.backward(xs[s], bs[s]))
        ref.apply_grads()
    np.testing.assert_allclose(r0["losses"], ref_losses, rtol=1e-13)
    np.testing.assert_allclose(r0["params"], ref.p, rtol=1e-10, atol=1e-13)
    np.testing.assert_allclose(r0["m1"], ref.m1, rtol=1e-10, atol=1e-15)
