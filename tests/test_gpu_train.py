"""GPU parity of batched training (forward, L1 loss, backward, Adam) against
the oracle.  The device computes in fp32 (tf32x3 on the tensor cores for
d = 16/32) with f64 reductions; tolerance per parameter tensor, norm-wise:
1e-4 for gradients (north_star's GNP bar), tighter for the loss."""
import os

import numpy as np
import pytest
from conftest import csr_of, f32, golden, rel_l2

pytestmark = pytest.mark.gpu


def slices(d, h, L):
    names, o = [], 0
    for nm, sz in [("enc1", h), ("enc1_b", h), ("enc2", h * d), ("enc2_b", d)]:
        names.append((nm, o, o + sz))
        o += sz
    for l in range(L):
        names.append((f"u{l}", o, o + d * d))
        o += d * d
        names.append((f"w{l}", o, o + d * d))
        o += d * d
    for nm, sz in [("dec1", d * h), ("dec1_b", h), ("dec2", h), ("dec2_b", 1)]:
        names.append((nm, o, o + sz))
        o += sz
    return names


def check_grads(got, want, dims, tol=1e-4):
    worst = 0.0
    for nm, a, b in slices(*dims):
        den = np.linalg.norm(want[a:b])
        if den == 0.0:
            assert np.linalg.norm(got[a:b]) <= 1e-12, nm
            continue
        e = np.linalg.norm(got[a:b] - want[a:b]) / den
        worst = max(worst, e)
        assert e <= tol, (nm, e)
    return worst


def dev_csr(capi, a):
    return capi.Csr.from_arrays(a.n, a.row_ptr, a.col_idx, a.values)


def test_small_batch_loss_and_grads(capi, cuda):
    g = golden("train_step.npz")  # dims (4, 8, 2): CUDA-core batched path
    a = csr_of("a", g)
    A = dev_csr(capi, a)
    m = capi.Model(A, (4, 8, 2), g["params"])
    t = capi.Trainer(m, 4)
    loss, grads, out = t.forward_backward(g["x"], g["b"])
    assert abs(loss - float(g["loss"])) <= 1e-5 * float(g["loss"])
    assert rel_l2(out, g["out"]) <= 1e-5
    check_grads(grads, g["grads"], (4, 8, 2))


def test_c1_batch_grads_tensor_cores(capi, oc, cuda):
    # d = 16: tcgen05 forward + backward layers, B = 4 on the C1 matrix
    g = golden("c1.npz")
    gs = golden("c1_train_step.npz")
    ah = oc.prescale(oc.gen_convection_diffusion(64, 0.0), 8.0)
    x, b = oc.gaussian_batch(ah, 3, 0, 4)
    A = dev_csr(capi, ah)
    m = capi.Model(A, (16, 32, 8), g["params"])
    t = capi.Trainer(m, 4)
    loss, grads, _ = t.forward_backward(x, b)
    assert abs(loss - float(gs["loss"])) <= 1e-5 * float(gs["loss"])
    check_grads(grads, gs["grads"], (16, 32, 8))


def test_d32_batch_grads_tensor_cores(capi, cuda):
    g = golden("c3_small_train_step.npz")  # d = 32, B = 8, var-coeff 24x24
    a = csr_of("a", g)
    m = capi.Model(dev_csr(capi, a), (32, 32, 8), g["params"])
    t = capi.Trainer(m, 8)
    loss, grads, _ = t.forward_backward(g["x"], g["b"])
    assert abs(loss - float(g["loss"])) <= 1e-5 * float(g["loss"])
    check_grads(grads, g["grads"], (32, 32, 8))


def test_adam_step_matches_oracle(capi, oc, cuda):
    g = golden("train_step.npz")
    a = csr_of("a", g)
    m = capi.Model(dev_csr(capi, a), (4, 8, 2), g["params"])
    t = capi.Trainer(m, 4, lr=1e-3)
    _, grads, _ = t.forward_backward(g["x"], g["b"])
    t.apply_grads()
    z = np.zeros_like(grads)
    want, m1w, m2w, _ = oc.adam_step((4, 8, 2), g["params"], grads, z, z, 0, 1e-3)
    assert np.allclose(t.params(), want, rtol=0, atol=1e-15 + 1e-13 * np.abs(want).max())
    m1, m2, step = t.adam_state()
    assert step == 1 and np.allclose(m1, m1w, atol=1e-18) and np.allclose(m2, m2w, rtol=1e-12)


def test_training_is_deterministic(capi, cuda):
    g = golden("train_step.npz")
    a = csr_of("a", g)
    runs = []
    for _ in range(2):
        m = capi.Model(dev_csr(capi, a), (4, 8, 2), g["params"])
        t = capi.Trainer(m, 4)
        runs.append([t.step(g["x"], g["b"]) for _ in range(5)] + list(t.params()))
    assert runs[0] == runs[1]


def test_train_preconditioner_tracks_reference(capi, oc, cuda):
    # reference train_preconditioner, Gaussian pairs only (spectral = 0), 20 steps
    g = golden("train_run.npz")
    a = oc.gen_convection_diffusion(6, 0.5)
    ah = oc.prescale(a, oc.gershgorin_gamma(a))
    best, losses, bl = capi.train_preconditioner(dev_csr(capi, ah), dims=(4, 8, 2), steps=20, batch=8,
                                                 spectral=0, arnoldi_m=10, seed=41, monitor_batch=8)
    want = g["losses"]
    assert abs(losses[0] - want[0]) <= 1e-5 * want[0]
    assert np.max(np.abs(losses - want) / want) <= 1e-3
    assert bl == min(losses) and bl < losses[0]
    assert rel_l2(best, g["best"]) <= 1e-3


def test_synthetic_steps_reduce_loss(capi, gnp, cuda):
    a = capi.Csr.generate("c3_varcoeff2d", 64, 2.0, 0.0, 2)
    ah = a.prescale(a.gamma())
    m = capi.Model(ah, (32, 32, 8), capi.init_params(32, 32, 8, 0))
    t = capi.Trainer(m, 8, lr=1e-3)
    losses = [t.step_synthetic(7) for _ in range(30)]
    assert all(np.isfinite(losses))
    assert np.mean(losses[-5:]) < np.mean(losses[:5])


def test_python_train_drop_in(gnp, cuda):
    a = gnp.prescale(gnp.gen_convection_diffusion(6, 0.5), 8.0)
    params, losses = gnp.train(a, steps=10, batch=8, spectral=0, arnoldi_m=10, seed=1, d=4, hidden=8,
                               layers=2)
    assert len(losses) == 11 and min(losses) <= losses[0]
    b = gnp.spmv(a, [1.0] * a.n)
    out = gnp.solve(a, b, precond="gnp", params=params, maxiters=200)
    assert out["status"] in ("converged", "maxiters")


def test_data_parallel_driver_single_rank_equals_step(capi, cuda):
    # paper_2406_00809_b200.dp on one rank (no process group): local backward,
    # (no-op) all-reduce, Adam — bit-identical to the fused trainer step
    import torch  # noqa: F401  (CUDA context for the zero-copy gradient view)
    from paper_2406_00809_b200.dp import DataParallelTrainer, TrainerEngine

    a = capi.Csr.generate("c3_varcoeff2d", 48, 2.0, 0.0, 2)
    ah = a.prescale(a.gamma())
    p0 = capi.init_params(32, 32, 8, 0)
    t1 = capi.Trainer(capi.Model(ah, (32, 32, 8), p0), 8, lr=1e-3)
    t2 = capi.Trainer(capi.Model(ah, (32, 32, 8), p0), 8, lr=1e-3)
    dp = DataParallelTrainer(TrainerEngine(t2))
    l1 = [t1.step_synthetic(11) for _ in range(4)]
    l2 = [dp.step_synthetic(11) for _ in range(4)]
    assert l1 == l2
    assert np.array_equal(t1.params(), t2.params())
    rng = np.random.default_rng(0)
    x = rng.standard_normal((ah.n, 8))
    b = np.stack([ah.spmv(x[:, k]) for k in range(8)], axis=1)
    assert dp.step(x, b) == t1.step(x.ravel(order="F"), b.ravel(order="F"))
    assert np.array_equal(t1.params(), t2.params())


@pytest.mark.parametrize("d,B", [(16, 3), (32, 6), (16, 128)])
def test_batch_sizes_vs_oracle(capi, oc, cuda, d, B):
    # B must divide 128 for the TMA training layers (3 and 6 take the
    # register-staged tcgen05 layer; 128 = one node per tile)
    a = oc.prescale(oc.gen_convection_diffusion(12, 0.4), 8.8).rounded_f32()
    dims = (d, 32, 3)
    p = f32(oc.init_params(*dims, 5))
    x, b = oc.gaussian_batch(a, 9, 0, B)
    want_loss, want = oc.batch_loss_grads(a, dims, p, x, b, B)
    m = capi.Model(dev_csr(capi, a), dims, p)
    t = capi.Trainer(m, B)
    loss, grads, _ = t.forward_backward(x, b)
    assert abs(loss - want_loss) <= 1e-5 * abs(want_loss)
    check_grads(grads, want, dims)


def test_tma_training_layers_match_fallback(capi, oc, cuda):
    # the same step through k_train_sell (default) and, in a subprocess with
    # GNPC_NO_TRAIN_SELL=1, through the register-staged tcgen05 layers
    import json
    import os
    import subprocess
    import sys

    code = r"""
import json, sys, numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
from paper_2406_00809_b200 import capi
import oracle
oc = oracle.restatement()
a = oc.prescale(oc.gen_convection_diffusion(20, 0.3), 8.6).rounded_f32()
p = oc.init_params(32, 32, 4, 2).astype(np.float32).astype(np.float64)
x, b = oc.gaussian_batch(a, 4, 0, 8)
A = capi.Csr.from_arrays(a.n, a.row_ptr, a.col_idx, a.values)
t = capi.Trainer(capi.Model(A, (32, 32, 4), p), 8)
loss, g, _ = t.forward_backward(x, b)
print(json.dumps({"loss": loss, "g": list(g)}))
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for off in ("0", "1"):
        env = dict(os.environ, GNPC_NO_TRAIN_SELL=off)
        r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert abs(outs[0]["loss"] - outs[1]["loss"]) <= 1e-6 * abs(outs[1]["loss"])
    g0, g1 = np.array(outs[0]["g"]), np.array(outs[1]["g"])
    assert np.linalg.norm(g0 - g1) <= 1e-4 * np.linalg.norm(g1)


@pytest.mark.parametrize("switch", ["GNPC_NO_PW_ENCODER", "GNPC_NO_DEC_TC"])
def test_encoder_decoder_paths_match_mlp_kernels(capi, oc, cuda, switch):
    # the piecewise-linear encoder (lift tables + interval sums) and the
    # tensor-core decoder against the CUDA-core MLP kernels they replace
    # (switched off in a subprocess), both against the oracle
    import json
    import os
    import subprocess
    import sys

    code = r"""
import json, sys, numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
from paper_2406_00809_b200 import capi
import oracle
oc = oracle.restatement()
a = oc.prescale(oc.gen_convection_diffusion(20, 0.3), 8.6).rounded_f32()
p = oc.init_params(32, 32, 3, 4).astype(np.float64)
p[32:64] = 0.3 * np.sin(np.arange(32))  # nonzero enc1 biases (flat order: enc1, enc1_b, ...): distinct kinks
p = p.astype(np.float32).astype(np.float64)
x, b = oc.gaussian_batch(a, 6, 0, 8)
A = capi.Csr.from_arrays(a.n, a.row_ptr, a.col_idx, a.values)
t = capi.Trainer(capi.Model(A, (32, 32, 3), p), 8)
loss, g, _ = t.forward_backward(x, b)
l2, g2 = oc.batch_loss_grads(a, (32, 32, 3), p, x, b, 8)
print(json.dumps({"loss": loss, "g": list(g), "want_loss": l2, "want": list(g2)}))
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for off in ("0", "1"):
        env = dict(os.environ, **{switch: off})
        r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    want = np.array(outs[0]["want"])
    for o in outs:
        assert abs(o["loss"] - o["want_loss"]) <= 1e-5 * abs(o["want_loss"])
        check_grads(np.array(o["g"]), want, (32, 32, 3))
    g0, g1 = np.array(outs[0]["g"]), np.array(outs[1]["g"])
    assert np.linalg.norm(g0 - g1) <= 1e-4 * np.linalg.norm(g1)


def test_piecewise_encoder_hidden64(capi, oc, cuda):
    # hidden 64 at d = 32: the interval sums run with 4 warps (128-row stages)
    a = oc.prescale(oc.gen_convection_diffusion(16, 0.3), 8.6).rounded_f32()
    dims = (32, 64, 2)
    p = oc.init_params(*dims, 6).astype(np.float64)
    p[64:128] = 0.2 * np.cos(np.arange(64))  # enc1 biases: distinct kinks
    p = f32(p)
    x, b = oc.gaussian_batch(a, 7, 0, 8)
    t = capi.Trainer(capi.Model(dev_csr(capi, a), dims, p), 8)
    loss, g, _ = t.forward_backward(x, b)
    want_loss, want = oc.batch_loss_grads(a, dims, p, x, b, 8)
    assert abs(loss - want_loss) <= 1e-5 * abs(want_loss)
    check_grads(g, want, dims)


def test_trained_model_refuses_apply_until_synced(capi, oc, cuda):
    # a trainer's Adam step rewrites the model's device operands but not its
    # host params / lift tables: applies must refuse the mixed state until
    # gnpc_trainer_sync_model, then match the oracle with the trained params
    a = oc.prescale(oc.gen_convection_diffusion(12, 0.4), 8.8).rounded_f32()
    dims = (16, 32, 3)
    p = f32(oc.init_params(*dims, 5))
    m = capi.Model(dev_csr(capi, a), dims, p)
    b = oc.gaussian_vector(2, a.n)
    m.apply(b)
    t = capi.Trainer(m, 4)
    x, bb = oc.gaussian_batch(a, 9, 0, 4)
    t.step(x, bb)
    with pytest.raises(capi.GnpcError):
        m.apply(b)
    t.sync_model()
    y = m.apply(b)
    want = oc.gnn_apply(a, dims, t.params(), b)
    assert rel_l2(y, want) <= 1e-4


@pytest.mark.parametrize("grid,tw", [(160, True), (157, True), (158, False)])
def test_training_strip_windows_match_csr_layers(capi, oc, cuda, grid, tw):
    # d = 32, B = 32 on var-coeff grids: 160^2 (25,600 nodes = 6,400 tiles of
    # 4 nodes, grid-line offset 40 tiles), 157^2 (offset 39 tiles + 1 node,
    # inside the one-node halo; a partial last tile) and 158^2 (39 tiles + 2
    # nodes: outside the halo, so the CSR layers run).  The training layers
    # over strip windows (node windows staged by TMA) against the CSR layers
    # (GNPC_NO_TW=1): each virtual row sums its node's entries in stored order
    # either way and the MMAs are the same, so loss and gradients are equal.
    a = oc.prescale(oc.gen_named("c3_varcoeff2d", grid, 2.0, 0.0, 2), 8.0).rounded_f32()
    dims = (32, 32, 8)
    p = f32(oc.init_params(*dims, 1))
    x, b = oc.gaussian_batch(a, 32, 0, 32)
    outs = []
    for off in ("0", "1"):
        os.environ["GNPC_NO_TW"] = off
        try:
            A = dev_csr(capi, a)
            t = capi.Trainer(capi.Model(A, dims, p), 32)
            loss, g, _ = t.forward_backward(x, b)
            flags = A.layout_flags()
            steps = [t.step(x, b) for _ in range(3)]
        finally:
            os.environ.pop("GNPC_NO_TW", None)
        assert bool(flags & 16) == (off == "0" and tw), flags
        outs.append((loss, np.array(g), steps))
    assert outs[0][0] == outs[1][0]
    assert np.array_equal(outs[0][1], outs[1][1])
    assert outs[0][2] == outs[1][2]
