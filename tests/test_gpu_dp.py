"""Data-parallel training on the CUDA trainer, world_size 2.

Two processes on cuda:0 exchange the flat f64 gradient over gloo (one GPU in
this environment; the collective is host-mediated, so neither rank's kernels
wait on the other's), each driving paper_2406_00809_b200.dp with the C-ABI
TrainerEngine on its half of every global batch.  Checks:
  * the two replicas stay bit-identical (params, Adam moments, losses);
  * they equal, bit for bit, one process that runs the same two half-batch
    trainers and averages their gradients before Adam (the all-reduce is
    the only difference);
  * they follow the single-process full-batch trajectory (the reference's
    accumulate over all columns, src/gnn.cpp:426-440) to rounding.
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

pytestmark = pytest.mark.gpu

DIMS = (32, 32, 4)
GLOBAL_B = 16
STEPS = 4


def problem():
    import oracle

    oc = oracle.restatement()
    a0 = oc.gen_named("c3_varcoeff2d", 32, 2.0, 0.0, 2)
    a = oc.prescale(a0, oc.gershgorin_gamma(a0)).rounded_f32()
    params = oc.init_params(*DIMS, 0).astype(np.float32).astype(np.float64)
    xs, bs = [], []
    for s in range(STEPS):
        x, b = oc.gaussian_batch(a, 7, s, GLOBAL_B)
        xs.append(x.reshape(GLOBAL_B, a.n).T.copy())
        bs.append(b.reshape(GLOBAL_B, a.n).T.copy())
    return a, params, xs, bs


def _trainer(capi, a, params, batch):
    A = capi.Csr.from_arrays(a.n, a.row_ptr, a.col_idx, a.values)
    return capi.Trainer(capi.Model(A, DIMS, params), batch, lr=1e-3), A


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2406_00809_b200 import capi
        from paper_2406_00809_b200.dp import DataParallelTrainer, TrainerEngine

        capi.check(capi.lib().gnpc_set_device(0))
        a, params, xs, bs = problem()
        t, _A = _trainer(capi, a, params, GLOBAL_B // world)
        dp = DataParallelTrainer(TrainerEngine(t))
        losses = [dp.step(xs[s], bs[s]) for s in range(STEPS)]
        m1, m2, step = t.adam_state()
        np.savez(f"{out}_{rank}.npz", params=t.params(), losses=np.array(losses), m1=m1, m2=m2)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_dp_world2_cuda_trainer(capi, cuda, tmp_path):
    import torch
    import torch.multiprocessing as mp

    from paper_2406_00809_b200.dp import TrainerEngine, shard_columns

    out = str(tmp_path / "dp")
    mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
    r0, r1 = np.load(f"{out}_0.npz"), np.load(f"{out}_1.npz")
    for k in ("params", "losses", "m1", "m2"):
        assert np.array_equal(r0[k], r1[k]), k

    # one process, the same two half-batch trainers, gradients averaged
    a, params, xs, bs = problem()
    half = GLOBAL_B // 2
    ts = [_trainer(capi, a, params, half) for _ in range(2)]
    es = [TrainerEngine(t) for t, _ in ts]
    losses = []
    for s in range(STEPS):
        ls = []
        for r, e in enumerate(es):
            cols = shard_columns(GLOBAL_B, r, 2)
            ls.append(e.backward(xs[s][:, cols], bs[s][:, cols]))
        torch.cuda.synchronize()
        g = es[0].grad_tensor() + es[1].grad_tensor()  # gloo's SUM of two ranks
        g.div_(2)
        for e in es:
            e.grad_tensor().copy_(g)
            e.apply_grads()
        losses.append((ls[0] + ls[1]) / 2)
    assert np.array_equal(np.array(losses), r0["losses"])
    assert np.array_equal(ts[0][0].params(), r0["params"])

    # and the single-process full-batch step (the reference's accumulate)
    t, _A = _trainer(capi, a, params, GLOBAL_B)
    full = [t.step(xs[s].ravel(order="F"), bs[s].ravel(order="F")) for s in range(STEPS)]
    # (the half-batch reductions round differently; Adam amplifies sign flips
    # of near-zero gradient components, hence the norm-wise bound)
    np.testing.assert_allclose(r0["losses"], full, rtol=1e-6)
    pf = t.params()
    assert np.linalg.norm(r0["params"] - pf) <= 1e-4 * np.linalg.norm(pf)
