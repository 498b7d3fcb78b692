"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Runs only in the build container (needs oracle/_ref/libgnpref.so, built by
`make -C oracle ref` from /root/reference).  The fixtures are committed so the
CPU pin tests and the GPU parity tests never touch /root/reference.

    python tests/golden/make_golden.py [--only spectral]
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402

MTX = "/root/reference/proj/tests/data/nonsym1138.mtx"


def f32(x):
    return np.asarray(x, np.float64).astype(np.float32).astype(np.float64)


def csr_dict(prefix, a):
    return {f"{prefix}_n": np.int64(a.n), f"{prefix}_row_ptr": a.row_ptr,
            f"{prefix}_col_idx": a.col_idx, f"{prefix}_values": a.values}


def spectral(R):
    """Spectral sampler + spectral-pair batch (src/sampler.cpp) on a 16x16
    convection-diffusion matrix, and a short spectral training run."""
    a = R.gen_convection_diffusion(16, 0.5)
    gam = R.gershgorin_gamma(a)
    ah = R.prescale(a, gam)
    s = R.spectral_sampler(ah, 20, 7)
    x, b = R.assemble_batch(ah, 20, 7, 9, 1, 8, 4)
    np.savez_compressed(os.path.join(HERE, "spectral.npz"), gamma=gam, m=20, seed=7, k=s["k"],
                        m_eff=s["m_eff"], s=s["s"], batch_seed=9, batch=8, spectral=4, x=x, b=b)
    c6 = R.gen_convection_diffusion(6, 0.5)
    c6h = R.prescale(c6, R.gershgorin_gamma(c6))
    best, losses, bl = R.train(c6h, (4, 8, 2), steps=20, batch=8, spectral=4, arnoldi_m=10, seed=41,
                               monitor_batch=8)
    np.savez_compressed(os.path.join(HERE, "train_run_spectral.npz"), best=best, losses=losses,
                        best_loss=bl)


def main():
    R = O.reference()
    if "--only" in sys.argv:
        assert sys.argv[sys.argv.index("--only") + 1] == "spectral"
        spectral(R)
        return
    out = {}

    # 1. the reference's only real-matrix fixture, parsed by the reference
    a = R.read_matrix_market(MTX)
    g = R.gershgorin_gamma(a)
    ah = R.prescale(a, g)
    np.savez_compressed(os.path.join(HERE, "nonsym1138.npz"), **csr_dict("a", a),
                        gamma=g, hash=np.uint64(R.csr_hash(a)), ahat_hash=np.uint64(R.csr_hash(ah)))
    # apply on it (fp32-rounded Â and params, as the device sees them)
    ah32 = ah.rounded_f32()
    p = R.init_params(16, 32, 8, 0)
    b = R.gaussian_vector(11, a.n)
    np.savez_compressed(os.path.join(HERE, "nonsym1138_apply.npz"), params32=f32(p), b=b,
                        out=R.gnn_apply(ah32, (16, 32, 8), f32(p), b))

    # 2. config C1: gen_convection_diffusion(64, 0) prescaled, seed-0 GNP, b ~ Rng(1)
    c1 = R.gen_convection_diffusion(64, 0.0)
    g1 = R.gershgorin_gamma(c1)
    c1h = R.prescale(c1, g1)
    p1 = R.init_params(16, 32, 8, 0)
    b1 = R.gaussian_vector(1, c1.n)
    np.savez_compressed(os.path.join(HERE, "c1.npz"), gamma=g1,
                        hash=np.uint64(R.csr_hash(c1)), ahat_hash=np.uint64(R.csr_hash(c1h)),
                        params=p1, b=b1, out=R.gnn_apply(c1h.rounded_f32(), (16, 32, 8), f32(p1), b1))
    s = R.fgmres(c1h, b1, maxiters=100, restart=10)
    np.savez_compressed(os.path.join(HERE, "c1_gmres.npz"), status=s["status"],
                        hist=np.array([h[:2] for h in s["history"]]), x=s["x"])

    # 3. small random matrix, odd dims (3, 4, 2): apply + backward
    sm = R.gen_random_nonsymmetric(200, 6, 1.5, 3)
    smh = R.prescale(sm, R.gershgorin_gamma(sm)).rounded_f32()
    ps = f32(R.init_params(3, 4, 2, 4))
    bs = R.gaussian_vector(5, 200)
    gs = R.gaussian_vector(6, 200)
    o, gr = R.gnn_forward_backward(smh, (3, 4, 2), ps, bs, gs)
    np.savez_compressed(os.path.join(HERE, "small_fwd_bwd.npz"), **csr_dict("a", smh), params=ps,
                        b=bs, gout=gs, out=o, grads=gr)

    # 4. training: one batch's loss + summed gradient + one Adam step (conv-diff 8)
    cd = R.gen_convection_diffusion(8, 0.3)
    cdh = R.prescale(cd, R.gershgorin_gamma(cd)).rounded_f32()
    dims = (4, 8, 2)
    pt = f32(R.init_params(*dims, 7))
    x, bb = R.gaussian_batch(cdh, 3, 0, 4)
    loss, grads, outb = R.batch_loss_grads(cdh, dims, pt, x, bb, 4, want_out=True)
    z = np.zeros_like(pt)
    p_after, m1, m2, t = R.adam_step(dims, pt, grads, z, z, 0, 1e-3)
    np.savez_compressed(os.path.join(HERE, "train_step.npz"), **csr_dict("a", cdh), params=pt,
                        x=x, b=bb, loss=loss, grads=grads, out=outb, p_after=p_after, m1=m1, m2=m2)
    # the same at d=16/h=32/L=8 on C1 (B=4)
    x1, b1b = R.gaussian_batch(c1h.rounded_f32(), 3, 0, 4)
    l1, g1b = R.batch_loss_grads(c1h.rounded_f32(), (16, 32, 8), f32(p1), x1, b1b, 4)
    np.savez_compressed(os.path.join(HERE, "c1_train_step.npz"), loss=l1, grads=g1b)

    # 5. trained preconditioner that converges (tests/test_gnn.cpp:393-413 setup)
    cv = R.gen_convection_diffusion(5, 0.2)
    cvh = R.prescale(cv, R.gershgorin_gamma(cv))
    best, losses, bl = R.train(cvh, (4, 8, 2), steps=30, batch=8, spectral=4, arnoldi_m=12,
                               seed=50, monitor_batch=16)
    bone = R.spmv(cvh, np.ones(cvh.n))
    sol = R.fgmres(cvh, bone, kind=1, dims=(4, 8, 2), params=best, maxiters=50)
    cvh32 = cvh.rounded_f32()
    bone32 = R.spmv(cvh32, np.ones(cvh.n))
    sol32 = R.fgmres(cvh32, bone32, kind=1, dims=(4, 8, 2), params=f32(best), maxiters=50)
    np.savez_compressed(os.path.join(HERE, "trained_conv5.npz"), params=best, losses=losses,
                        best_loss=bl, status=sol["status"],
                        hist=np.array([h[:2] for h in sol["history"]]),
                        status32=sol32["status"], hist32=np.array([h[:2] for h in sol32["history"]]))
    # a well-trained, fast-converging case (12 vs 32 GMRES iterations): iteration
    # parity +-1 is meaningful here, unlike the 50-iteration case above which moves
    # by ~10 iterations under any 1e-7 perturbation of M
    c8 = R.gen_convection_diffusion(8, 0.3)
    c8h = R.prescale(c8, R.gershgorin_gamma(c8))
    best8, losses8, bl8 = R.train(c8h, (8, 16, 4), steps=600, batch=8, spectral=4, arnoldi_m=12,
                                  seed=50, monitor_batch=16)
    c8h32 = c8h.rounded_f32()
    b8 = R.spmv(c8h32, np.ones(c8h.n))
    s8 = R.fgmres(c8h32, b8, kind=1, dims=(8, 16, 4), params=f32(best8), maxiters=100, restart=20)
    np.savez_compressed(os.path.join(HERE, "trained_conv8.npz"), params=best8, losses=losses8,
                        status=s8["status"], hist=np.array([h[:2] for h in s8["history"]]))
    # 6. a short reference training run with Gaussian pairs only (spectral = 0)
    c6 = R.gen_convection_diffusion(6, 0.5)
    c6h = R.prescale(c6, R.gershgorin_gamma(c6))
    best6, losses6, bl6 = R.train(c6h, (4, 8, 2), steps=20, batch=8, spectral=0, arnoldi_m=10,
                                  seed=41, monitor_batch=8)
    np.savez_compressed(os.path.join(HERE, "train_run.npz"), best=best6, losses=losses6, best_loss=bl6)
    # 7. one batch at d=32 (tcgen05 width) on a variable-coefficient 2D problem
    import ctypes  # noqa: F401
    sys.path.insert(0, ROOT)
    from paper_2406_00809_b200 import capi

    cv = capi.Csr.generate("c3_varcoeff2d", 24, 2.0, 0.0, 2)
    rp, ci, v = cv.arrays()
    c3 = O.Csr(cv.n, rp, ci, v)
    c3h = R.prescale(c3, R.gershgorin_gamma(c3)).rounded_f32()
    p3 = f32(R.init_params(32, 32, 8, 0))
    x3, b3 = R.gaussian_batch(c3h, 3, 0, 8)
    l3, g3 = R.batch_loss_grads(c3h, (32, 32, 8), p3, x3, b3, 8)
    np.savez_compressed(os.path.join(HERE, "c3_small_train_step.npz"), **csr_dict("a", c3h), params=p3,
                        x=x3, b=b3, loss=l3, grads=g3)
    spectral(R)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
