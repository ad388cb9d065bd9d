"""GPU parity: the CUDA path through the C-ABI (libgwas.so) vs the CPU oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star): max |b_gpu - b_ref| / SE_ref <= 1e-8, max Var relative error <= 1e-8,
statuses identical.  Invariance checks (block size, input placement, X_R dtype, trait slicing) are bitwise.
"""
import ctypes as C

import numpy as np
import pytest

import datagen
import oracle
from gpu_helpers import TOL_B, TOL_VAR, compare

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _gw():
    import paper_1207_2169_b200 as gw
    return gw


def _ld(n, es=1):
    q = 16 // es
    return (n + q - 1) // q * q


def _run(cfg, ds, XR, **kw):
    gw = _gw()
    eng = gw.Gwas(cfg.n, cfg.p, cfg.t, device=0, **kw)
    eng.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2)
    b, v, s = eng.run(XR)
    torch.cuda.synchronize()
    out = b.cpu().numpy(), v.cpu().numpy(), s.cpu().numpy()
    eng.close()
    return out


@pytest.fixture(scope="module")
def c0():
    cfg = datagen.CONFIGS[0]
    ds = datagen.dataset(cfg)
    XR = datagen.xr_dosages(cfg, ld=_ld(cfg.n))
    ref = oracle.gls_sequence(ds.Phi, ds.XL, XR[:, :cfg.n].T.astype(np.float64), ds.Y, ds.h2, ds.s2)
    return cfg, ds, XR, ref


# ------------------------------------------------------------------ K1/K2 kernel unit checks
@pytest.mark.parametrize("M,N,K,u8,nsq", [(300, 200, 1000, True, None), (129, 131, 17, False, None),
                                          (1, 8, 16, False, None), (257, 300, 333, False, 160),
                                          (8192, 136, 1000, True, None), (64, 500, 4096, False, 256),
                                          (8192, 1500, 300, True, None), (8000, 1300, 99, False, 640)])
def test_gemm_kernel_vs_fp64_reference(M, N, K, u8, nsq):
    gw = _gw()
    rng = np.random.default_rng(M * 7 + N)
    if u8:
        A = rng.integers(0, 3, size=(M, _ld(K, 1)), dtype=np.uint8)
    else:
        A = rng.standard_normal((M, _ld(K, 8)))
    B = rng.standard_normal((N, _ld(K, 8)))
    Ct = gw.gemm_tn(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), nsq=nsq, K=K).cpu().numpy()
    Af = A[:, :K].astype(np.float64)
    Bf = B[:, :K]
    ref = Af @ Bf.T
    if nsq is not None:
        ref[:, nsq:] = (Af * Af) @ Bf[nsq:].T
        scale = (np.abs(Af) ** 2).max() * np.abs(Bf).max() * K
    else:
        scale = np.abs(Af).max() * np.abs(Bf).max() * K
    err = np.max(np.abs(Ct - ref)) / scale
    assert err <= 1e-15, err


# ------------------------------------------------------------------ config 0: every pair
def test_c0_all_pairs(c0):
    cfg, ds, XR, ref = c0
    b, v, s = _run(cfg, ds, torch.from_numpy(XR).cuda(), block_cols=cfg.block_cols)
    eb, ev = compare(b, v, s, ref)
    print(f"C0 all {cfg.m * cfg.t} pairs: max|db|/SE={eb:.3e} max Var rel={ev:.3e}")
    assert eb <= TOL_B and ev <= TOL_VAR


def test_c0_full_output_mode(c0):
    cfg, ds, XR, ref = c0
    b, v, s = _run(cfg, ds, torch.from_numpy(XR).cuda(), output_mode="full")
    assert b.shape == (cfg.m, cfg.t, cfg.p + 1)
    eb, ev = compare(b, v, s, ref, full=True)
    assert eb <= TOL_B and ev <= TOL_VAR, (eb, ev)


def test_c0_literal_var_convention(c0):
    cfg, ds, XR, _ = c0
    ref = oracle.gls_sequence(ds.Phi, ds.XL, XR[:500, :cfg.n].T.astype(np.float64), ds.Y, ds.h2, ds.s2,
                              var_convention=1)
    b, v, s = _run(cfg, ds, torch.from_numpy(XR[:500]).cuda(), var_convention="literal")
    eb, ev = compare(b, v, s, ref)
    assert eb <= TOL_B and ev <= TOL_VAR, (eb, ev)


# ------------------------------------------------------------------ invariances (bitwise)
def test_block_size_and_placement_invariance(c0):
    cfg, ds, XR, _ = c0
    dev = torch.from_numpy(XR).cuda()
    base = _run(cfg, ds, dev, block_cols=2000)
    for k in (512, 333, 8192, 1):
        other = _run(cfg, ds, dev[:600] if k == 1 else dev, block_cols=k)
        for x, y in zip(base, other):
            np.testing.assert_array_equal(x[: y.shape[0]], y)
    # pinned host input: 1-D staging copy (ld % 16 == 0) and 2-D staging copy (ld = n)
    other = _run(cfg, ds, dev, block_cols=300, overlap=True)   # two-stream block pipelining
    for x, y in zip(base, other):
        np.testing.assert_array_equal(x, y)
    host_pad = torch.from_numpy(XR).pin_memory()
    host_n = torch.from_numpy(np.ascontiguousarray(XR[:, :cfg.n])).pin_memory()
    for src in (host_pad, host_n):
        other = _run(cfg, ds, src, block_cols=700)
        for x, y in zip(base, other):
            np.testing.assert_array_equal(x, y)


def test_f64_dosages_equal_u8(c0):
    cfg, ds, XR, _ = c0
    base = _run(cfg, ds, torch.from_numpy(XR).cuda())
    XRf = torch.from_numpy(XR[:, :cfg.n].astype(np.float64)).cuda()  # ld = n = 200 (even): 16-byte rows
    other = _run(cfg, ds, XRf, xr_dtype="f64")
    for x, y in zip(base, other):
        np.testing.assert_array_equal(x, y)


def test_trait_slice_equals_single_trait(c0):
    cfg, ds, XR, _ = c0
    dev = torch.from_numpy(XR).cuda()
    full = _run(cfg, ds, dev)
    j = 2
    cfg1 = datagen.custom_config(n=cfg.n, p=cfg.p, m=cfg.m, t=1)
    ds1 = datagen.Dataset(cfg1, ds.Phi, ds.XL, np.asfortranarray(ds.Y[:, [j]]), ds.h2[[j]], ds.s2[[j]])
    one = _run(cfg1, ds1, dev)
    np.testing.assert_array_equal(full[0][:, j], one[0][:, 0])
    np.testing.assert_array_equal(full[1][:, j], one[1][:, 0])


# ------------------------------------------------------------------ ragged shapes, edge cases
@pytest.mark.parametrize("n,p,t,m,k", [(333, 3, 37, 777, 256), (17, 2, 1, 40, 16), (129, 6, 9, 300, 300),
                                       (250, 1, 3, 130, 64)])
def test_ragged_shapes_f64(n, p, t, m, k):
    cfg = datagen.custom_config(n=n, p=p, m=m, t=t, index=200 + n)
    ds = datagen.dataset(cfg)
    G = datagen.xr_dosages(cfg).astype(np.float64)
    ld = _ld(n, 8)
    XR = np.zeros((m, ld))
    XR[:, :n] = G
    ref = oracle.gls_sequence(ds.Phi, ds.XL, G.T, ds.Y, ds.h2, ds.s2)
    b, v, s = _run(cfg, ds, torch.from_numpy(XR).cuda(), xr_dtype="f64", block_cols=k, output_mode="full")
    eb, ev = compare(b, v, s, ref, full=True)
    assert eb <= TOL_B and ev <= TOL_VAR, (eb, ev)


def test_collinear_and_nonfinite_pairs():
    cfg = datagen.custom_config(n=120, p=4, m=50, t=3, index=301)
    ds = datagen.dataset(cfg)
    G = datagen.xr_dosages(cfg).astype(np.float64)
    G[0] = 1.0                      # monomorphic: a multiple of the intercept
    G[1] = 3.0 * ds.XL[:, 1]        # copy of a covariate
    G[2] = 2.0 * ds.XL[:, -1]       # copy of the sex column
    ref = oracle.gls_sequence(ds.Phi, ds.XL, G.T, ds.Y, ds.h2, ds.s2)
    assert (ref["status"][:3] == oracle.STATUS_COLLINEAR).all()
    G2 = G.copy()
    G2[3, 7] = np.nan               # non-finite dosage
    b, v, s = _run(cfg, ds, torch.from_numpy(G2).cuda(), xr_dtype="f64")
    assert (s[:3] == 1).all() and (s[3] == 2).all() and (s[4:] == 0).all()
    assert np.isnan(b[:4]).all() and np.isnan(v[:4]).all()
    eb, ev = compare(b[4:], v[4:], s[4:], {k: (x[4:] if k != "traits" else x) for k, x in ref.items()})
    assert eb <= TOL_B and ev <= TOL_VAR


def test_empty_and_single_column(c0):
    cfg, ds, XR, ref = c0
    gw = _gw()
    eng = gw.Gwas(cfg.n, cfg.p, cfg.t, device=0)
    eng.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2)
    dev = torch.from_numpy(XR).cuda()
    b, v, s = eng.run(dev[:0])
    assert b.shape == (0, cfg.t)
    b, v, s = eng.run(dev[5:6])
    torch.cuda.synchronize()
    eb, ev = compare(b.cpu().numpy(), v.cpu().numpy(), s.cpu().numpy(),
                     {k: (x[5:6] if k != "traits" else x) for k, x in ref.items()})
    assert eb <= TOL_B and ev <= TOL_VAR
    eng.close()


def test_setup_errors():
    gw = _gw()
    cfg = datagen.custom_config(n=64, p=3, m=10, t=2, index=302)
    ds = datagen.dataset(cfg)
    eng = gw.Gwas(cfg.n, cfg.p, cfg.t, device=0)
    with pytest.raises(gw.GwasError) as e:
        eng.setup(ds.Phi, ds.XL, ds.Y, np.array([0.5, 1.5]), ds.s2)
    assert e.value.code == 1 and "h2[1]" in str(e.value)
    with pytest.raises(gw.GwasError) as e:
        eng.setup(ds.Phi, ds.XL, ds.Y, ds.h2, np.array([1.0, 0.0]))
    assert e.value.code == 1
    XL = ds.XL.copy()
    XL[:, 2] = XL[:, 1]
    with pytest.raises(gw.GwasError) as e:
        eng.setup(ds.Phi, XL, ds.Y, ds.h2, ds.s2)
    assert e.value.code == 2 and "trait 0" in str(e.value)
    # h2 = 1 with the (singular, Phi 1 = 0) sample-centred GRM: D_j has a non-positive denominator (reading A7)
    with pytest.raises(gw.GwasError) as e:
        eng.setup(ds.Phi, ds.XL, ds.Y, np.array([0.3, 1.0]), ds.s2)
    assert e.value.code == 2 and "trait 1" in str(e.value)
    with pytest.raises(gw.GwasError):
        gw.Gwas(3, 5, 1)
    eng.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2)  # a failed setup leaves the engine usable
    with pytest.raises(gw.GwasError) as e:        # pageable host X_R is refused (would serialise staging)
        import paper_1207_2169_b200._lib as L
        XR = np.zeros((4, 64), dtype=np.uint8)
        b, v, s = eng.alloc_outputs(4)
        L.check(L.lib.gwas_run(eng._ctx, 4, XR.ctypes.data, 64, b.data_ptr(), v.data_ptr(), s.data_ptr()))
    assert e.value.code == 1
    # the round-2 queries: run configuration, and estimation diagnostics only on an estimation context
    import ctypes as C
    import paper_1207_2169_b200._lib as L
    info = eng.run_info()
    assert info["block_cols"] == 8192 and info["fused_k2"] is True   # t (p + 2) = 10 <= 28: K2 in K1's epilogue
    gs = np.zeros(cfg.t, dtype=np.int32)
    assert L.lib.gwas_estimate_grid_argmax(eng._ctx, gs.ctypes.data_as(C.POINTER(C.c_int32))) == L.GWAS_E_STATE
    assert L.lib.gwas_run_info(None, None, None) == L.GWAS_E_STATE
    eng.close()


def test_attach_after_state_copy(c0):
    """Multi-GPU replication path on one device: a second context attaches to a byte copy of the state."""
    cfg, ds, XR, _ = c0
    gw = _gw()
    a = gw.Gwas(cfg.n, cfg.p, cfg.t, device=0)
    a.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2)
    bcopy = gw.Gwas(cfg.n, cfg.p, cfg.t, device=0)
    bcopy.state.copy_(a.state)
    bcopy.attach()
    dev = torch.from_numpy(XR).cuda()
    r1 = [x.cpu().numpy() for x in a.run(dev)]
    r2 = [x.cpu().numpy() for x in bcopy.run(dev)]
    for x, y in zip(r1, r2):
        np.testing.assert_array_equal(x, y)
    wrong = gw.Gwas(cfg.n, cfg.p, cfg.t + 1, device=0)
    with pytest.raises(gw.GwasError) as e:
        wrong.attach()
    assert e.value.code in (6,)


@pytest.mark.parametrize("i8,lr,t", [(8, 0, 40), (0, -1, 40), (8, -1, 40), (8, 0, 4)])
def test_attach_after_state_copy_modes(i8, lr, t):
    """Attached contexts (the other ranks of a multi-GPU run) read every run-time choice made at setup from the
    state header (int8 digit layout, low-rank rank and operand widths): results bitwise equal to the setup rank."""
    gw = _gw()
    cfg = datagen.custom_config(n=160, p=3, m=500, t=t, index=460 + t)
    ds = datagen.dataset(cfg)
    XR = torch.from_numpy(datagen.xr_dosages(cfg, ld=_ld(cfg.n))).cuda()
    a = gw.Gwas(cfg.n, cfg.p, cfg.t, device=0, int8_slices=i8, trait_rank=lr, block_cols=200)
    a.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2)
    bcopy = gw.Gwas(cfg.n, cfg.p, cfg.t, device=0, int8_slices=i8, trait_rank=lr, block_cols=200, overlap=True)
    bcopy.state.copy_(a.state)
    bcopy.attach()
    assert bcopy.trait_rank() == a.trait_rank()
    r1 = [x.cpu().numpy() for x in a.run(XR)]
    r2 = [x.cpu().numpy() for x in bcopy.run(XR)]
    for x, y in zip(r1, r2):
        np.testing.assert_array_equal(x, y)
    ref = oracle.gls_sequence(ds.Phi, ds.XL, XR[:, :cfg.n].cpu().numpy().T.astype(np.float64), ds.Y, ds.h2, ds.s2)
    eb, ev = compare(*r2, ref)
    assert eb <= TOL_B and ev <= TOL_VAR


# ------------------------------------------------------------------ int8-sliced mode
@pytest.mark.parametrize("S", [8, 7])
def test_int8_sliced_c0_all_pairs(c0, S):
    cfg, ds, XR, ref = c0
    b, v, s = _run(cfg, ds, torch.from_numpy(XR).cuda(), int8_slices=S)
    eb, ev = compare(b, v, s, ref)
    print(f"C0 int8-sliced all pairs: max|db|/SE={eb:.3e} max Var rel={ev:.3e}")
    assert eb <= TOL_B and ev <= TOL_VAR


@pytest.mark.parametrize("S", [8, 7])
def test_int8_sliced_full_mode_and_invariance(c0, S):
    cfg, ds, XR, ref = c0
    dev = torch.from_numpy(XR).cuda()
    b, v, s = _run(cfg, ds, dev, int8_slices=S, output_mode="full")
    eb, ev = compare(b, v, s, ref, full=True)
    assert eb <= TOL_B and ev <= TOL_VAR, (eb, ev)
    base = _run(cfg, ds, dev, int8_slices=S)
    for k in (333, 1):
        other = _run(cfg, ds, dev[:300] if k == 1 else dev, int8_slices=S, block_cols=k)
        for x, y in zip(base, other):
            np.testing.assert_array_equal(x[: y.shape[0]], y)
    other = _run(cfg, ds, torch.from_numpy(XR).pin_memory(), int8_slices=S, block_cols=700)
    for x, y in zip(base, other):
        np.testing.assert_array_equal(x, y)
    other = _run(cfg, ds, dev, int8_slices=S, block_cols=256, overlap=True)   # two-stream block pipelining
    for x, y in zip(base, other):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("S", [8, 7])
@pytest.mark.parametrize("n,p,t,m,k", [(333, 3, 37, 777, 256), (17, 2, 1, 40, 16), (129, 6, 70, 300, 300),
                                       (1000, 4, 200, 1000, 512)])
def test_int8_sliced_ragged(n, p, t, m, k, S):
    cfg = datagen.custom_config(n=n, p=p, m=m, t=t, index=400 + n)
    ds = datagen.dataset(cfg)
    XR = datagen.xr_dosages(cfg, ld=_ld(n))
    ref = oracle.gls_sequence(ds.Phi, ds.XL, XR[:, :n].T.astype(np.float64), ds.Y, ds.h2, ds.s2)
    b, v, s = _run(cfg, ds, torch.from_numpy(XR).cuda(), int8_slices=S, block_cols=k)
    eb, ev = compare(b, v, s, ref)
    assert eb <= TOL_B and ev <= TOL_VAR, (eb, ev)


def test_int8_sliced_rejects_f64_dosages():
    gw = _gw()
    with pytest.raises(gw.GwasError):
        gw.Gwas(64, 3, 2, device=0, xr_dtype="f64", int8_slices=8)
    with pytest.raises(gw.GwasError):
        gw.Gwas(64, 3, 2, device=0, int8_slices=6)


# ------------------------------------------------------------------ guard bands (compute-sanitizer is closed on this pool)
@pytest.mark.parametrize("i8,ovl,mode", [(0, False, "snp"), (8, True, "full"), (0, True, "full"), (8, False, "snp")])
def test_no_writes_outside_caller_buffers(i8, ovl, mode):
    """Every buffer the library writes (state, workspace, b, var, status) sits between sentinel guard bands;
    after setup + a ragged multi-block run from device and from pinned host memory the bands are intact."""
    import ctypes as C
    import paper_1207_2169_b200._lib as L
    cfg = datagen.custom_config(n=333, p=3, m=700, t=37, index=501)
    ds = datagen.dataset(cfg)
    XR = datagen.xr_dosages(cfg, ld=_ld(cfg.n))
    o = L.default_options()
    o.int8_slices, o.overlap, o.block_cols = i8, 1 if ovl else 0, 256
    o.output_mode = L.OUT_FULL if mode == "full" else L.OUT_SNP
    n, p, t, m = cfg.n, cfg.p, cfg.t, cfg.m
    sb = L.lib.gwas_state_bytes(n, p, t, C.byref(o))
    wb = L.lib.gwas_workspace_bytes(n, p, t, C.byref(o))
    G = 1 << 16
    per = (p + 1) if mode == "full" else 1

    def guarded(nbytes):
        buf = torch.full((nbytes + 2 * G,), 0xA5, dtype=torch.uint8, device="cuda")
        return buf, buf[G:G + nbytes]

    state_g, state = guarded(sb)
    work_g, work = guarded(wb)
    b_g, b = guarded(m * t * per * 8)
    v_g, v = guarded(m * t * per * 8)
    s_g, s = guarded(m * t)
    ctx = C.c_void_p()
    h2, s2 = np.ascontiguousarray(ds.h2), np.ascontiguousarray(ds.s2)
    phi, xl, y = np.ascontiguousarray(ds.Phi), np.asfortranarray(ds.XL), np.asfortranarray(ds.Y)  # kept alive
    L.check(L.lib.gwas_setup(C.byref(o), n, p, t, phi.ctypes.data, xl.ctypes.data, y.ctypes.data, h2.ctypes.data,
                             s2.ctypes.data, state.data_ptr(), sb, work.data_ptr(), wb, C.byref(ctx)))
    xd = torch.from_numpy(XR).cuda()
    xh = torch.from_numpy(XR).pin_memory()
    for src in (xd, xh):
        L.check(L.lib.gwas_run(ctx, m, src.data_ptr(), XR.shape[1], b.data_ptr(), v.data_ptr(), s.data_ptr()))
    torch.cuda.synchronize()
    L.lib.gwas_destroy(ctx)
    for g in (state_g, work_g, b_g, v_g, s_g):
        assert bool((g[:G] == 0xA5).all()) and bool((g[-G:] == 0xA5).all())
    # and the results are still right
    ref = oracle.gls_sequence(ds.Phi, ds.XL, XR[:, :n].T.astype(np.float64), ds.Y, ds.h2, ds.s2)
    bb = b.view(torch.float64).reshape(m, t, *((per,) if mode == "full" else ())).cpu().numpy()
    vv = v.view(torch.float64).reshape(m, t, *((per,) if mode == "full" else ())).cpu().numpy()
    ss = s.view(torch.int8).reshape(m, t).cpu().numpy()
    eb, ev = compare(bb, vv, ss, ref, full=(mode == "full"))
    assert eb <= TOL_B and ev <= TOL_VAR


@pytest.mark.parametrize("S", [8, 7])
def test_int8_sliced_kernel_variants_agree(c0, S):
    """The 1-SM (cluster 1, 2, 4) and 2-SM (cta_group::2; one or two pairs per cluster, persistent or not) int8
    kernels, with 64- or 128-byte K stages, give bitwise identical results (the int32 digit products are exact, the
    fp64 recombination is the same code)."""
    import os
    import subprocess
    import sys
    code = ("import sys, numpy as np, torch, datagen; sys.path.insert(0, 'tests');"
            "import paper_1207_2169_b200 as gw;"
            "cfg = datagen.custom_config(n=333, p=3, m=5000, t=37, index=601); ds = datagen.dataset(cfg);"
            "X = torch.from_numpy(datagen.xr_dosages(cfg, ld=336)).cuda();"
            f"e = gw.Gwas(cfg.n, cfg.p, cfg.t, int8_slices={S}, block_cols=4096); e.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2);"
            "b, v, s = e.run(X); torch.cuda.synchronize();"
            "np.save(sys.argv[1], np.stack([b.cpu().numpy(), v.cpu().numpy()]))")
    outs = []
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        # the 4096-row block has 16 x 9 pair tiles (8 x 9 two-pair tiles), more than the co-resident clusters, so the
        # persistent 2-SM kernel loops over several tiles per cluster; persist 0 = one cluster per tile
        variants = [(k, cl, bk, ps) for bk in ("128", "64") for k, cl in (("1sm", "1"), ("1sm", "2"), ("1sm", "4"),
                    ("2sm", "2"), ("2sm", "4")) for ps in ("1", "0") if k == "2sm" or ps == "1"]
        for i, (kern, cl, bk, ps) in enumerate(variants):
            f = os.path.join(d, f"r{i}.npy")
            env = dict(os.environ, GWAS_I8_KERNEL=kern, GWAS_I8_CLUSTER=cl, GWAS_I8_BK=bk, GWAS_I8_PERSIST=ps)
            subprocess.run([sys.executable, "-c", code, f], check=True, env=env, cwd=os.path.dirname(os.path.dirname(__file__)))
            outs.append(np.load(f))
    for o in outs[1:]:
        np.testing.assert_array_equal(outs[0], o)


@pytest.mark.parametrize("i8", [0, 8])
def test_split_k_skinny_products(i8):
    """n >= 4096 with few traits: the skinny K2 / K2b products are split along K (fixed ranges, fixed-order sum)."""
    cfg = datagen.custom_config(n=4100, p=2, m=300, t=3, index=700)
    ds = datagen.dataset(cfg)
    XR = datagen.xr_dosages(cfg, ld=_ld(cfg.n))
    ref = oracle.gls_sequence(ds.Phi, ds.XL, XR[:, :cfg.n].T.astype(np.float64), ds.Y, ds.h2, ds.s2)
    b, v, s = _run(cfg, ds, torch.from_numpy(XR).cuda(), int8_slices=i8, block_cols=128)
    eb, ev = compare(b, v, s, ref)
    assert eb <= TOL_B and ev <= TOL_VAR, (eb, ev)
    b2, v2, s2 = _run(cfg, ds, torch.from_numpy(XR).cuda(), int8_slices=i8, block_cols=300, overlap=True)
    np.testing.assert_array_equal(b, b2)
    np.testing.assert_array_equal(v, v2)


# ------------------------------------------------------------------ CLAK-Chol single-trait path (Alg. 3, NEXT-1)
@pytest.mark.parametrize("i8,n,mode,k", [(0, 200, "snp", 2000), (8, 200, "full", 512), (0, 333, "full", 256),
                                         (8, 333, "snp", 100), (0, 4100, "snp", 256), (8, 4100, "snp", 300)])
def test_chol_single_trait(i8, n, mode, k):
    cfg = datagen.custom_config(n=n, p=4, m=600 if n < 1000 else 200, t=1, index=800 + n)
    ds = datagen.dataset(cfg)
    XR = datagen.xr_dosages(cfg, ld=_ld(n))
    ref = oracle.gls_sequence(ds.Phi, ds.XL, XR[:, :n].T.astype(np.float64), ds.Y, ds.h2, ds.s2)
    b, v, s = _run(cfg, ds, torch.from_numpy(XR).cuda(), algorithm="chol", int8_slices=i8, output_mode=mode,
                   block_cols=k)
    eb, ev = compare(b, v, s, ref, full=(mode == "full"))
    print(f"chol n={n} int8={i8}: max|db|/SE={eb:.3e} max Var rel={ev:.3e}")
    assert eb <= TOL_B and ev <= TOL_VAR, (eb, ev)
    if mode == "snp":   # block size / overlap invariance (bitwise)
        b2, v2, s2 = _run(cfg, ds, torch.from_numpy(XR).cuda(), algorithm="chol", int8_slices=i8, block_cols=k + 37,
                          overlap=True)
        np.testing.assert_array_equal(b, b2)
        np.testing.assert_array_equal(v, v2)


def test_chol_errors():
    gw = _gw()
    with pytest.raises(gw.GwasError) as e:
        gw.Gwas(64, 3, 2, device=0, algorithm="chol")
    assert e.value.code == 1
    cfg = datagen.custom_config(n=64, p=3, m=10, t=1, index=802)
    ds = datagen.dataset(cfg)
    eng = gw.Gwas(cfg.n, cfg.p, cfg.t, device=0, algorithm="chol")
    with pytest.raises(gw.GwasError) as e:   # h2 = 1 with the singular sample-centred GRM: M not SPD
        eng.setup(ds.Phi, ds.XL, ds.Y, np.array([1.0]), ds.s2)
    assert e.value.code == 2
    eng.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2)
    eng.close()


@pytest.mark.parametrize("i8,ovl,mode", [(0, False, "snp"), (0, True, "full"), (8, True, "snp")])
def test_host_outputs_stream_back(c0, i8, ovl, mode):
    """Pinned host outputs (per-block D2H on the library's stream) equal device outputs bitwise."""
    cfg, ds, XR, _ = c0
    gw = _gw()
    eng = gw.Gwas(cfg.n, cfg.p, cfg.t, device=0, int8_slices=i8, overlap=ovl, output_mode=mode, block_cols=300)
    eng.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2)
    dev = [x.cpu().numpy() for x in eng.run(torch.from_numpy(XR).cuda())]
    host = eng.alloc_outputs(cfg.m, host=True)
    eng.run(torch.from_numpy(XR).pin_memory(), out=host)
    torch.cuda.synchronize()
    for x, y in zip(dev, host):
        np.testing.assert_array_equal(x, y.numpy())
    mixed = (host[0], host[1], torch.empty((cfg.m, cfg.t), dtype=torch.int8, device="cuda"))
    with pytest.raises(gw.GwasError):
        eng.run(torch.from_numpy(XR).cuda(), out=mixed)
    eng.close()


# ------------------------------------------------------------------ NEXT-2: K2 fused into K1's epilogue
@pytest.mark.parametrize("i8,alg,n,p,t,k", [(0, "eig", 200, 4, 4, 2000), (0, "eig", 333, 5, 4, 256), (0, "eig", 300, 6, 4, 256),
                                            (8, "eig", 200, 4, 4, 512), (8, "eig", 517, 3, 8, 300),
                                            (0, "chol", 333, 4, 1, 256), (8, "chol", 200, 5, 1, 700),
                                            (0, "eig", 1000, 4, 1, 8192)])
def test_fused_k2_matches_oracle_and_unfused(i8, alg, n, p, t, k):
    """Few traits: K2 contracted in K1's epilogue (fuse_k2, default) vs the separate K2 product and the oracle.
    t (p + 2) = 28 at (333, 5, 4) is the FP64 fusion limit (32 at (300, 6, 4): unfused); (517, 3, 8) the int8 one."""
    cfg = datagen.custom_config(n=n, p=p, m=900, t=t, index=400 + n + t)
    ds = datagen.dataset(cfg)
    XR = datagen.xr_dosages(cfg, ld=_ld(n))
    ref = oracle.gls_sequence(ds.Phi, ds.XL, XR[:, :n].T.astype(np.float64), ds.Y, ds.h2, ds.s2)
    dev = torch.from_numpy(XR).cuda()
    fused = _run(cfg, ds, dev, block_cols=k, int8_slices=i8, algorithm=alg, overlap=True)
    plain = _run(cfg, ds, dev, block_cols=k, int8_slices=i8, algorithm=alg, fuse_k2=False)
    for res in (fused, plain):
        eb, ev = compare(*res, ref)
        assert eb <= TOL_B and ev <= TOL_VAR, (eb, ev)
    np.testing.assert_array_equal(fused[2], plain[2])
    # the fused path is itself bitwise invariant to the block size
    other = _run(cfg, ds, dev, block_cols=128, int8_slices=i8, algorithm=alg)
    for x, y in zip(fused, other):
        np.testing.assert_array_equal(x, y)


# ------------------------------------------------------------------ low-rank trait weights (reading L1)
@pytest.mark.parametrize("i8,mode,ovl", [(0, "snp", False), (0, "full", True), (8, "snp", True), (8, "full", False)])
def test_lowrank_trait_weights(i8, mode, ovl):
    """trait_rank = -1: K2 against U_r of D = U S V^T (r << t) + the K = r recombination, vs the oracle's exact GLS."""
    gw = _gw()
    cfg = datagen.custom_config(n=240, p=4, m=700, t=96, index=451)
    ds = datagen.dataset(cfg)
    XR = datagen.xr_dosages(cfg, ld=_ld(cfg.n))
    ref = oracle.gls_sequence(ds.Phi, ds.XL, XR[:, :cfg.n].T.astype(np.float64), ds.Y, ds.h2, ds.s2)
    eng = gw.Gwas(cfg.n, cfg.p, cfg.t, device=0, block_cols=256, int8_slices=i8, output_mode=mode, overlap=ovl,
                  trait_rank=-1)
    eng.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2)
    r, s0, sr = eng.trait_rank()
    assert 8 <= r <= 40 and sr <= 1e-15 * s0, (r, s0, sr)
    b, v, s = eng.run(torch.from_numpy(XR).cuda())
    torch.cuda.synchronize()
    res = (b.cpu().numpy(), v.cpu().numpy(), s.cpu().numpy())
    eng.close()
    eb, ev = compare(*res, ref, full=mode == "full")
    print(f"low-rank r={r} (i8={i8}, {mode}): max|db|/SE={eb:.2e} Var rel={ev:.2e}")
    assert eb <= TOL_B and ev <= TOL_VAR
    # a state copy attaches with the chosen rank; results identical
    exact = _run(cfg, ds, torch.from_numpy(XR).cuda(), block_cols=256, int8_slices=i8, output_mode=mode)
    np.testing.assert_array_equal(exact[2], res[2])


def test_lowrank_skipped_for_few_traits():
    gw = _gw()
    cfg = datagen.custom_config(n=100, p=3, m=10, t=8, index=452)
    ds = datagen.dataset(cfg)
    eng = gw.Gwas(cfg.n, cfg.p, cfg.t, device=0, trait_rank=-1)
    eng.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2)
    assert eng.trait_rank()[0] == 0
    eng.close()


# ------------------------------------------------------------------ maximum sizes and degenerate cases
@pytest.mark.parametrize("i8,mode", [(0, "full"), (7, "full"), (8, "snp")])
def test_max_covariates_p12(i8, mode):
    """p = 12 (the largest X_L width the kernels are instantiated for), ragged n, several blocks."""
    cfg = datagen.custom_config(n=301, p=12, m=520, t=9, index=470)
    ds = datagen.dataset(cfg)
    XR = datagen.xr_dosages(cfg, ld=_ld(cfg.n))
    ref = oracle.gls_sequence(ds.Phi, ds.XL, XR[:, :cfg.n].T.astype(np.float64), ds.Y, ds.h2, ds.s2)
    b, v, s = _run(cfg, ds, torch.from_numpy(XR).cuda(), int8_slices=i8, output_mode=mode, block_cols=200)
    eb, ev = compare(b, v, s, ref, full=mode == "full")
    assert eb <= TOL_B and ev <= TOL_VAR, (eb, ev)


def test_degenerate_h2_zero_and_identity_kinship():
    """h2 = 0 (M = sigma2 I for any Phi) and Phi = I (M = sigma2 I for any h2): the GLS reduces to OLS.  Checked
    against numpy lstsq (independent of both the oracle and the GPU path), plus the oracle."""
    cfg = datagen.custom_config(n=150, p=3, m=200, t=4, index=471)
    ds = datagen.dataset(cfg)
    XR = datagen.xr_dosages(cfg, ld=_ld(cfg.n))
    G = XR[:, :cfg.n].T.astype(np.float64)
    for Phi, h2 in ((ds.Phi, np.zeros(cfg.t)), (np.eye(cfg.n), ds.h2)):
        b, v, s = _run(cfg, datagen.Dataset(cfg, Phi, ds.XL, ds.Y, h2, ds.s2), torch.from_numpy(XR).cuda())
        for j in range(cfg.t):
            for i in (0, 57, cfg.m - 1):
                X = np.column_stack([ds.XL, G[:, i]])
                beta, res, *_ = np.linalg.lstsq(X, ds.Y[:, j], rcond=None)
                var_g = np.linalg.inv(X.T @ X)[-1, -1] * ds.s2[j]   # Var = (X^T M^-1 X)^-1 with M = s2 I
                assert abs(b[i, j] - beta[-1]) <= 1e-9 * np.sqrt(var_g)
                assert abs(v[i, j] - var_g) <= 1e-9 * var_g
        ref = oracle.gls_sequence(Phi, ds.XL, G, ds.Y, h2, ds.s2)
        eb, ev = compare(b, v, s, ref)
        assert eb <= TOL_B and ev <= TOL_VAR


def test_sigma2_scaling_on_gpu():
    """sigma2 -> alpha sigma2: b unchanged, Var x alpha (textbook convention, reading A1); bitwise-close."""
    cfg = datagen.custom_config(n=180, p=4, m=300, t=5, index=472)
    ds = datagen.dataset(cfg)
    XR = torch.from_numpy(datagen.xr_dosages(cfg, ld=_ld(cfg.n))).cuda()
    b1, v1, s1 = _run(cfg, ds, XR)
    b2, v2, s2 = _run(cfg, datagen.Dataset(cfg, ds.Phi, ds.XL, ds.Y, ds.h2, 4.0 * ds.s2), XR)
    np.testing.assert_array_equal(s1, s2)
    np.testing.assert_allclose(b2, b1, rtol=1e-12, atol=0)
    np.testing.assert_allclose(v2, 4.0 * v1, rtol=1e-12)


@pytest.mark.parametrize("i8", [0, 7])
def test_lowrank_more_traits_than_individuals(i8):
    """t > n (the paper's omics scenario C has t up to 1e5 at n = 1e3): D^T is factored instead of D."""
    gw = _gw()
    cfg = datagen.custom_config(n=120, p=3, m=400, t=300, index=473)
    ds = datagen.dataset(cfg)
    XR = datagen.xr_dosages(cfg, ld=_ld(cfg.n))
    ref = oracle.gls_sequence(ds.Phi, ds.XL, XR[:, :cfg.n].T.astype(np.float64), ds.Y, ds.h2, ds.s2)
    eng = gw.Gwas(cfg.n, cfg.p, cfg.t, device=0, block_cols=256, int8_slices=i8, trait_rank=-1)
    eng.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2)
    r, s0, sr = eng.trait_rank()
    assert 8 <= r <= 40 and sr <= 1e-15 * s0, (r, s0, sr)
    b, v, s = eng.run(torch.from_numpy(XR).cuda())
    torch.cuda.synchronize()
    res = (b.cpu().numpy(), v.cpu().numpy(), s.cpu().numpy())
    eng.close()
    eb, ev = compare(*res, ref)
    print(f"low-rank t > n: r={r} max|db|/SE={eb:.2e} Var rel={ev:.2e}")
    assert eb <= TOL_B and ev <= TOL_VAR


@pytest.mark.parametrize("lr", [0, -1])
def test_many_traits_beyond_grid_limit(lr):
    """t (p + 2) > 65535 operand rows (grid-stride setup kernels), checked on a seeded subset of traits."""
    cfg = datagen.custom_config(n=64, p=2, m=96, t=16500, index=474)
    ds = datagen.dataset(cfg)
    XR = datagen.xr_dosages(cfg, ld=_ld(cfg.n))
    b, v, s = _run(cfg, ds, torch.from_numpy(XR).cuda(), block_cols=64, trait_rank=lr)
    traits = np.unique(np.concatenate([[0, cfg.t - 1], np.random.default_rng(0).choice(cfg.t, 30, replace=False)]))
    ref = oracle.gls_sequence(ds.Phi, ds.XL, XR[:, :cfg.n].T.astype(np.float64), ds.Y, ds.h2, ds.s2, traits=traits)
    eb, ev = compare(b[:, traits], v[:, traits], s[:, traits], ref)
    assert eb <= TOL_B and ev <= TOL_VAR, (eb, ev)


def test_lowrank_fused_k3_matches_unfused():
    """The fused recombination + Schur kernel against the separate K = r products + K3 (GWAS_LR_UNFUSED=1), and
    both against the oracle (full output mode, t = 78 not a multiple of the 32-trait tile, ragged SNP block; the
    separate products need even t)."""
    import os
    import subprocess
    import sys
    code = ("import sys, numpy as np, torch, datagen; sys.path.insert(0, 'tests');"
            "import paper_1207_2169_b200 as gw;"
            "cfg = datagen.custom_config(n=200, p=4, m=333, t=78, index=475); ds = datagen.dataset(cfg);"
            "X = torch.from_numpy(datagen.xr_dosages(cfg, ld=208)).cuda();"
            "e = gw.Gwas(cfg.n, cfg.p, cfg.t, trait_rank=-1, block_cols=150, output_mode='full');"
            "e.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2); b, v, s = e.run(X); torch.cuda.synchronize();"
            "np.savez(sys.argv[1], b=b.cpu().numpy(), v=v.cpu().numpy(), s=s.cpu().numpy(), r=e.trait_rank()[0])")
    import tempfile
    outs = []
    with tempfile.TemporaryDirectory() as d:
        for i, unfused in enumerate((False, True)):
            f = os.path.join(d, f"r{i}.npz")
            env = dict(os.environ)
            if unfused:
                env["GWAS_LR_UNFUSED"] = "1"
            subprocess.run([sys.executable, "-c", code, f], check=True, env=env,
                           cwd=os.path.dirname(os.path.dirname(__file__)))
            outs.append(np.load(f))
    assert outs[0]["r"] > 0
    cfg = datagen.custom_config(n=200, p=4, m=333, t=78, index=475)
    ds = datagen.dataset(cfg)
    XR = datagen.xr_dosages(cfg, ld=208)
    ref = oracle.gls_sequence(ds.Phi, ds.XL, XR[:, :cfg.n].T.astype(np.float64), ds.Y, ds.h2, ds.s2)
    for o in outs:
        eb, ev = compare(o["b"], o["v"], o["s"], ref, full=True)
        assert eb <= TOL_B and ev <= TOL_VAR, (eb, ev)
    np.testing.assert_array_equal(outs[0]["s"], outs[1]["s"])


# ------------------------------------------------------------------ K3 on the trait-tiled K2 output (t >= 32)
@pytest.mark.parametrize("n,p,t,m,k,mode,var", [(200, 5, 300, 700, 256, "snp", "literal"),
                                                (150, 12, 40, 300, 128, "full", "textbook"),
                                                (120, 1, 129, 333, 200, "full", "literal"),
                                                (64, 5, 20000, 50, 32, "snp", "textbook")])
def test_trait_tiled_k3(n, p, t, m, k, mode, var):
    """Many traits, FP64 exact weights: K2 writes C trait-tiled (ctile.cuh) and K3 streams it with bulk copies
    (schur_solve_tma): aligned row ranges (t = 40 .. 300) and flattened trait-block ranges (t = 2e4, 157 trait
    blocks), p = 1 / 5 / 12, SNP and full output, both Var conventions, a monomorphic SNP (status 1, NaN payload),
    ragged trait blocks (t % 128 != 0) and ragged row tiles -- vs the oracle."""
    cfg = datagen.custom_config(n=n, p=p, m=m, t=t, index=900 + p + t)
    ds = datagen.dataset(cfg)
    XR = datagen.xr_dosages(cfg, ld=_ld(n)).copy()
    XR[3, :] = 1                         # SNP 3 monomorphic: collinear with the intercept
    ref = oracle.gls_sequence(ds.Phi, ds.XL, XR[:, :n].T.astype(np.float64), ds.Y, ds.h2, ds.s2,
                              var_convention=1 if var == "literal" else 0)
    assert (ref["status"][3] == oracle.STATUS_COLLINEAR).all()
    b, v, s = _run(cfg, ds, torch.from_numpy(XR).cuda(), block_cols=k, output_mode=mode, var_convention=var,
                   overlap=True)
    eb, ev = compare(b, v, s, ref, full=mode == "full")
    print(f"tiled K3 n={n} p={p} t={t} {mode}/{var}: max|db|/SE={eb:.2e} Var rel={ev:.2e}")
    assert eb <= TOL_B and ev <= TOL_VAR, (eb, ev)


# ------------------------------------------------------------------ block_cols = 0 (auto)
@pytest.mark.parametrize("n,p,t,m", [(17, 2, 1, 40), (333, 3, 37, 777), (200, 4, 4, 2000), (1000, 4, 1000, 300)])
def test_auto_block_size(n, p, t, m):
    """block_cols = 0: the library picks k (a multiple of 128 in [4096, 16384], reported by gwas_run_info) from the
    wave quantisation of K1/K2; results are bitwise those of a fixed k and match the oracle."""
    gw = _gw()
    cfg = datagen.custom_config(n=n, p=p, m=m, t=t, index=950 + n + t)
    ds = datagen.dataset(cfg)
    XR = datagen.xr_dosages(cfg, ld=_ld(n))
    dev = torch.from_numpy(XR).cuda()
    eng = gw.Gwas(n, p, t, device=0, block_cols=0, overlap=True)
    eng.setup(ds.Phi, ds.XL, ds.Y, ds.h2, ds.s2)
    info = eng.run_info()
    assert 4096 <= info["block_cols"] <= 16384 and info["block_cols"] % 128 == 0
    b, v, s = eng.run(dev)
    torch.cuda.synchronize()
    auto = (b.cpu().numpy(), v.cpu().numpy(), s.cpu().numpy())
    eng.close()
    fixed = _run(cfg, ds, dev, block_cols=96)
    for x, y in zip(auto, fixed):
        np.testing.assert_array_equal(x, y)
    ref = oracle.gls_sequence(ds.Phi, ds.XL, XR[:, :n].T.astype(np.float64), ds.Y, ds.h2, ds.s2)
    eb, ev = compare(*auto, ref)
    assert eb <= TOL_B and ev <= TOL_VAR, (eb, ev)


@pytest.mark.parametrize("i8", [0, 8])
def test_minimum_n_square_design(i8):
    """n = w = p + 1 (the smallest n the problem admits): every X_i is square, the GLS solution interpolates,
    b = X_i^-1 y_j and Var = X_i^-1 M_j X_i^-T (pin P8 of the oracle) -- through every kernel at its smallest shape."""
    p = 4
    n = p + 1
    cfg = datagen.custom_config(n=n, p=p, m=64, t=3, S=64, index=990)
    ds = datagen.dataset(cfg)
    XR = datagen.xr_dosages(cfg, ld=_ld(n))
    ref = oracle.gls_sequence(ds.Phi, ds.XL, XR[:, :n].T.astype(np.float64), ds.Y, ds.h2, ds.s2)
    b, v, s = _run(cfg, ds, torch.from_numpy(XR).cuda(), int8_slices=i8, block_cols=16)
    np.testing.assert_array_equal(s, ref["status"])
    eb, ev = compare(b, v, s, ref)
    # square systems amplify rounding by cond(X_i); the tolerance stays the north star's
    assert eb <= TOL_B and ev <= TOL_VAR, (eb, ev)
