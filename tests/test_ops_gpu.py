"""GPU parity of the full-FFT / projection / update / solver operators against
the reference (oracle/_ref: verbatim fft.cpp, solver.cpp, scan.cpp, simulate.cpp)."""
import numpy as np
import pytest

from conftest import DATA, cnormal, rel_l2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2408_03532_b200")


@pytest.mark.parametrize("shape", [(64, 64), (256, 256), (512, 512), (32, 128), (8, 16)])
def test_fft2_ifft2_c128(ref, shape):
    rng = np.random.default_rng(11)
    z = cnormal(rng, (2,) + shape)
    f = P.fast_fft2(torch.from_numpy(z).cuda()).cpu().numpy()
    fi = P.fast_ifft2(torch.from_numpy(z).cuda()).cpu().numpy()
    for b in range(2):
        assert rel_l2(f[b], ref.fast_fft2(z[b])) <= 1e-13
        assert rel_l2(fi[b], ref.fast_ifft2(z[b])) <= 1e-13


def test_fft2_c64():
    rng = np.random.default_rng(12)
    z = cnormal(rng, (3, 512, 512), np.complex64)
    f = P.fast_fft2(torch.from_numpy(z).cuda()).cpu().numpy()
    assert rel_l2(f, np.fft.fft2(z.astype(np.complex128))) <= 1e-6


def test_fft_known_answers():
    z = np.zeros((4, 4), np.complex128)
    z[0, 0] = 1
    assert np.allclose(P.fast_fft2(torch.from_numpy(z).cuda()).cpu().numpy(), 1)
    c = np.full((4, 4), 2.5 + 0j)
    f = P.fast_fft2(torch.from_numpy(c).cuda()).cpu().numpy()
    assert abs(f[0, 0] - 40) < 1e-12 and np.abs(f.ravel()[1:]).max() < 1e-12


@pytest.mark.parametrize("dtype,tol", [(np.complex128, 1e-12), (np.complex64, 1e-5)])
def test_project_modulus(ref, dtype, tol):
    rng = np.random.default_rng(13)
    x = cnormal(rng, (256, 256), dtype)
    d = np.abs(cnormal(rng, (256, 256))) * 10
    d = d.astype(np.float64 if dtype == np.complex128 else np.float32)
    got = P.project_modulus(torch.from_numpy(x).cuda(), torch.from_numpy(d).cuda()).cpu().numpy()
    want = ref.project_modulus(x.astype(np.complex128), d.astype(np.float64))
    assert rel_l2(got, want) <= tol


def test_project_modulus_fixed_point_and_zero():
    rng = np.random.default_rng(14)
    x = cnormal(rng, (64, 64))
    d = np.abs(np.fft.fft2(x))
    got = P.project_modulus(torch.from_numpy(x).cuda(), torch.from_numpy(d).cuda()).cpu().numpy()
    assert rel_l2(got, x) <= 1e-10
    z = np.zeros((64, 64), np.complex128)
    got0 = P.project_modulus(torch.from_numpy(z).cuda(), torch.from_numpy(d).cuda()).cpu().numpy()
    assert rel_l2(got0, np.fft.ifft2(d)) <= 1e-12


@pytest.mark.parametrize("dtype,tol", [(np.complex128, 1e-10), (np.complex64, 1e-5)])
def test_band_residual(ref, dtype, tol):
    g = P.pft_plan_2d(256, 256, 32, 32, 32, 32, 1e-3)
    r = ref.RefPlan.create(DATA / "scope_table_v1.txt", 256, 256, 32, 32, 32, 32, 1e-3)
    rng = np.random.default_rng(15)
    x = cnormal(rng, (256, 256), dtype)
    dcrop = (np.abs(cnormal(rng, (64, 64))) * 50).astype(np.float64)
    got = P.band_residual(g, torch.from_numpy(x).cuda(), torch.from_numpy(dcrop).cuda())
    want = r.band_residual(x.astype(np.complex128), dcrop.astype(np.float32 if dtype == np.complex64 else np.float64))
    assert rel_l2(got.cpu().numpy(), want) <= tol


def test_updates_and_windows(ref):
    rng = np.random.default_rng(16)
    z, pr, pj = (cnormal(rng, (32, 32)) for _ in range(3))
    zt = torch.from_numpy(z.copy()).cuda()
    P.pie_object_update(zt, torch.from_numpy(pr).cuda(), torch.from_numpy(pj).cuda(), 0.7)
    assert rel_l2(zt.cpu().numpy(), ref.pie_object_update(z, pr, pj, 0.7)) <= 1e-15
    pt = torch.from_numpy(pr.copy()).cuda()
    P.epie_probe_update(pt, torch.from_numpy(z).cuda(), torch.from_numpy(pj).cuda(), 0.3, True)
    assert rel_l2(pt.cpu().numpy(), ref.epie_probe_update(pr, z, pj, 0.3)) <= 1e-15
    with pytest.raises(RuntimeError):
        P.epie_probe_update(pt, torch.from_numpy(z).cuda(), torch.from_numpy(pj).cuda(), 0.3, False)
    frame = cnormal(rng, (100, 90))
    offs = np.array([[0, 0], [3, 7], [68, 58]])
    pat = P.window_slice(torch.from_numpy(frame).cuda(), offs, 32, 32).cpu().numpy()
    for k, (r0, c0) in enumerate(offs):
        assert np.array_equal(pat[k], frame[r0:r0 + 32, c0:c0 + 32])
    ft = torch.from_numpy(frame.copy()).cuda()
    P.set_window(ft, (3, 7), torch.from_numpy(z).cuda())
    f2 = frame.copy()
    f2[3:35, 7:39] = z
    assert np.array_equal(ft.cpu().numpy(), f2)


def test_objective_value(ref):
    rng = np.random.default_rng(17)
    frame = cnormal(rng, (160, 160))
    probe = cnormal(rng, (64, 64))
    offs = np.array([[r, c] for r in (0, 48, 96) for c in (0, 48, 96)])
    d = np.abs(cnormal(rng, (9, 64, 64))) * 30
    got = P.objective_value(torch.from_numpy(frame).cuda(), torch.from_numpy(probe).cuda(), offs,
                            torch.from_numpy(d).cuda())
    want = ref.objective_value(frame, probe, offs, d)
    assert abs(got - want) / want <= 1e-12


def _small_problem(rng, n=128, w=64, npos=9):
    obj = (0.5 + 0.5 * rng.random((n, n))) * np.exp(1j * rng.uniform(-1, 1, (n, n)))
    yy, xx = np.mgrid[0:w, 0:w] - (w - 1) / 2
    probe = np.exp(-(xx ** 2 + yy ** 2) / (2 * (w / 5) ** 2)) * np.exp(1j * 0.3 * (xx ** 2 + yy ** 2) / w ** 2)
    k = int(round(np.sqrt(npos)))
    pos = np.linspace(0, n - w, k).round().astype(int)
    offs = np.array([[r, c] for r in pos for c in pos], np.int64)
    return obj.astype(np.complex128), probe.astype(np.complex128), offs


@pytest.mark.parametrize("blind", [False, True])
def test_hybrid_solve_c128_matches_reference(ref, blind):
    rng = np.random.default_rng(18)
    obj, probe, offs = _small_problem(rng)
    d = ref.simulate(obj, probe, offs)
    init = np.exp(1j * 0.1 * rng.standard_normal(obj.shape)) * 0.8
    pinit = probe * 0.9
    kw = dict(pft_sweeps=2, fft_sweeps=2, beta=1.0, gamma=1.0, beta_pft=1.0 / 64 ** 2,
              gamma_pft=1.0 / 64 ** 2, eps_pft=1e-3, blind=blind)
    f_ref, p_ref, obj_ref, _, _ = ref.hybrid_solve(init, pinit, offs, d, table_path=DATA / "scope_table_v1.txt",
                                                   **kw)
    cfg = P.SolverConfig(**kw)
    res = P.hybrid_solve(d, offs, pinit, init, cfg, dtype=np.complex128)
    assert res.sweeps_run == 4
    assert rel_l2(res.frame, f_ref) <= 1e-9
    assert rel_l2(res.probe, p_ref) <= 1e-9
    assert np.allclose(res.objective, obj_ref, rtol=1e-8)


@pytest.mark.parametrize("tv", [(0.05, 0.0), (0.03, 0.02)])
def test_hybrid_solve_tv_c128_matches_reference(ref, tv):
    """TV step per sweep (solver.cpp:264-279) on the GPU (k_tv) against the
    verbatim reference solver: band + FFT sweeps, blind."""
    rng = np.random.default_rng(28)
    obj, probe, offs = _small_problem(rng)
    d = ref.simulate(obj, probe, offs)
    init = np.exp(1j * 0.1 * rng.standard_normal(obj.shape)) * 0.8
    pinit = probe * 0.9
    kw = dict(pft_sweeps=2, fft_sweeps=2, beta=1.0, gamma=1.0, beta_pft=1.0 / 64 ** 2,
              gamma_pft=1.0 / 64 ** 2, eps_pft=1e-3, blind=True)
    f_ref, p_ref, obj_ref, _, _ = ref.hybrid_solve(init, pinit, offs, d, table_path=DATA / "scope_table_v1.txt",
                                                   tv_mag=tv[0], tv_phase=tv[1], **kw)
    cfg = P.SolverConfig(tv_lambda_mag=tv[0], tv_lambda_phase=tv[1], **kw)
    res = P.hybrid_solve(d, offs, pinit, init, cfg, dtype=np.complex128)
    assert rel_l2(res.frame, f_ref) <= 1e-9
    assert rel_l2(res.probe, p_ref) <= 1e-9
    assert np.allclose(res.objective, obj_ref, rtol=1e-8)
    res32 = P.hybrid_solve(d, offs, pinit, init, cfg, dtype=np.complex64)
    from oracle import pft_oracle as O
    tab = O.load_scope_table(DATA / "scope_table_v1.txt")
    ff, _, _ = O.hybrid_solve(init, pinit, offs, d, table=tab, dtype=np.complex64, tv_mag=tv[0],
                              tv_phase=tv[1], **kw)
    assert rel_l2(res32.frame, f_ref) <= 4.0 * rel_l2(ff, f_ref) + 1e-6


# complex64 ePIE gate: the GPU complex64 solve may deviate from
# the reference (double) by at most EPIE_FLOOR_FACTOR x the deviation of
# oracle<float> -- the reference's algorithm run entirely in complex64
# (oracle/pft_oracle.hybrid_solve(dtype=complex64)) -- on the same problem,
# measured inside each test, plus an absolute slack for the tiny-divergence case.
# Factor: measured on the full cfg3 problem (1 band + 1 FFT sweep, 800 sequential
# updates; tools/epie_floor_ratio.py) the streaming band kernels land at 3.7 / 3.9 x
# the floor (frame / probe), the axis-reordered ones (eval_band.cu) at 4.9 / 5.6 x:
# two samples of complex64 rounding in different summation orders.
EPIE_FLOOR_FACTOR = 6.0


def _epie_float_floor(init, pinit, offs, d, f_ref, p_ref, **kw):
    from oracle import pft_oracle as O
    tab = O.load_scope_table(DATA / "scope_table_v1.txt")
    ff, pf, _ = O.hybrid_solve(init, pinit, offs, d, table=tab, dtype=np.complex64, **kw)
    return rel_l2(ff, f_ref), rel_l2(pf, p_ref)


def _epie_gate(floor):
    return EPIE_FLOOR_FACTOR * floor + 1e-6


def test_hybrid_solve_c64_tracks_reference(ref):
    rng = np.random.default_rng(19)
    obj, probe, offs = _small_problem(rng)
    d = ref.simulate(obj, probe, offs)
    init = np.exp(1j * 0.1 * rng.standard_normal(obj.shape)) * 0.8
    kw = dict(pft_sweeps=2, fft_sweeps=3, beta=1.0, gamma=1.0, beta_pft=1.0 / 64 ** 2,
              gamma_pft=1.0 / 64 ** 2, eps_pft=1e-3, blind=True)
    f_ref, p_ref, obj_ref, _, _ = ref.hybrid_solve(init, probe, offs, d, table_path=DATA / "scope_table_v1.txt",
                                                   **kw)
    ff, fp = _epie_float_floor(init, probe, offs, d, f_ref, p_ref, **kw)
    res = P.hybrid_solve(d, offs, probe, init, P.SolverConfig(**kw), dtype=np.complex64)
    ef, ep = rel_l2(res.frame, f_ref), rel_l2(res.probe, p_ref)
    assert ef <= _epie_gate(ff), (ef, ff)
    assert ep <= _epie_gate(fp), (ep, fp)


def test_evaluator_band_and_fft(ref):
    rng = np.random.default_rng(20)
    obj, probe, offs = _small_problem(rng, n=160, w=64, npos=9)
    d = ref.simulate(obj, probe, offs)
    g = P.pft_plan_2d(64, 64, 8, 8, 8, 8, 1e-3)
    r = ref.RefPlan.create(DATA / "scope_table_v1.txt", 64, 64, 8, 8, 8, 8, 1e-3)
    dcrop = np.stack([ref.crop_centered(dj, 8, 8) for dj in d])
    fs, bs = P.evaluate(torch.from_numpy(obj).cuda(), torch.from_numpy(probe).cuda(), offs,
                        torch.from_numpy(d).cuda(), plan=g, d_crop=torch.from_numpy(dcrop).cuda())
    assert abs(fs / 9 - ref.objective_value(obj, probe, offs, d)) <= 1e-10 * max(1.0, fs)
    want_b = 0.0
    for j, (r0, c0) in enumerate(offs):
        ex = probe * obj[r0:r0 + 64, c0:c0 + 64]
        want_b += np.sum((np.abs(r.apply(ex)) - dcrop[j]) ** 2)
    assert abs(bs - want_b) <= 1e-9 * max(want_b, 1e-30) + 1e-18


def test_cfg3_full_problem_one_band_one_fft_sweep(ref):
    """BASELINE configs[2] problem (1024^2 object, 400 positions of 256^2, M=64),
    blind, stable steps: GPU c128 == reference hybrid_solve to 1e-10 after one
    PFT sweep + one FFT sweep; c64 within EPIE_FLOOR_FACTOR x the oracle<float>
    divergence (float rounding through 800 sequential dependent updates)."""
    from paper_2408_03532_b200 import problems as PR
    prob = PR.make_problem("cfg3", seed=0)
    n, w = prob.obj.shape[0], prob.probe.shape[0]
    rng = np.random.default_rng(1)
    init = rng.random((n, n)) * np.exp(1j * rng.random((n, n)) * np.pi / 2)
    pinit = PR.make_probe(w, 48.0, "cuda").abs().to(torch.complex128).cpu().numpy()
    d = prob.d.cpu().numpy().astype(np.float64)
    kw = dict(pft_sweeps=1, fft_sweeps=1, beta=0.5, gamma=0.05, beta_pft=0.25 / w ** 2,
              gamma_pft=0.25 * 0.05 / w ** 2, eps_pft=1e-3, blind=True)
    fr, pr, objr, _, flags = ref.hybrid_solve(init, pinit, prob.offsets, d, mt=32,
                                              table_path=DATA / "scope_table_v1.txt", **kw)
    assert flags == 0
    r128 = P.hybrid_solve(d, prob.offsets, pinit, init, P.SolverConfig(mt1=32, mt2=32, **kw),
                          dtype=np.complex128)
    assert rel_l2(r128.frame, fr) <= 1e-10 and rel_l2(r128.probe, pr) <= 1e-10
    assert np.allclose(r128.objective, objr, rtol=1e-10)
    r64 = P.hybrid_solve(d, prob.offsets, pinit, init, P.SolverConfig(mt1=32, mt2=32, **kw))
    ff, fp = _epie_float_floor(init, pinit, prob.offsets, d, fr, pr, mt=32, **kw)
    ef, ep = rel_l2(r64.frame, fr), rel_l2(r64.probe, pr)
    assert ef <= _epie_gate(ff) and ep <= _epie_gate(fp), (ef, ff, ep, fp)



@pytest.mark.parametrize("w,dtype,pft", [(64, np.complex128, 1), (128, np.complex128, 0), (64, np.complex64, 1),
                                         (256, np.complex64, 0), (512, np.complex64, 1)])
def test_hybrid_solve_shuffled_matches_reference(ref, w, dtype, pft):
    """Shuffled visit order (the reference's mt19937_64 Fisher-Yates stream,
    solver.cpp:164-169) through the band and full-FFT stages, blind. w = 512
    complex64 runs the radix-8 register FFT stage and objective (eval_fft.cuh)."""
    rng = np.random.default_rng(31)
    obj, probe, offs = _small_problem(rng, n=2 * w + 32, w=w, npos=9)
    d = ref.simulate(obj, probe, offs)
    init = np.exp(1j * 0.1 * rng.standard_normal(obj.shape)) * 0.8
    kw = dict(pft_sweeps=pft, fft_sweeps=2, beta=0.5, gamma=0.05, beta_pft=0.25 / w ** 2,
              gamma_pft=0.0125 / w ** 2, eps_pft=1e-3, blind=True, shuffled=True, seed=7)
    got = P.hybrid_solve(d, offs, probe * 0.9, init, P.SolverConfig(**kw), dtype=dtype)
    f_ref, p_ref, _, _, _ = ref.hybrid_solve(init, probe * 0.9, offs, d, table_path=DATA / "scope_table_v1.txt",
                                             **kw)
    ef, ep = rel_l2(got.frame, f_ref), rel_l2(got.probe, p_ref)
    if dtype == np.complex128:
        assert ef <= 1e-10 and ep <= 1e-10
    else:
        ff, fp = _epie_float_floor(init, probe * 0.9, offs, d, f_ref, p_ref, **kw)
        assert ef <= _epie_gate(ff) and ep <= _epie_gate(fp), (ef, ff, ep, fp)


def test_evaluator_tma_windows_c64(ref):
    """cfg4/cfg5 window shape (512^2, band M=128, p=64): the TMA rows pass reads
    scan windows at even and odd complex64 offsets (8-byte phase shift) and
    multiplies the probe in-kernel; band and FFT sums vs the reference."""
    rng = np.random.default_rng(22)
    w, n = 512, 600
    obj = (cnormal(rng, (n, n)) * 0.5).astype(np.complex64)
    probe = cnormal(rng, (w, w)).astype(np.complex64)
    offs = np.array([[0, 0], [3, 5], [17, 64], [88, 87], [41, 2]], np.int64)
    d = np.abs(cnormal(rng, (len(offs), w, w))).astype(np.float32) * 20
    g = P.pft_plan_2d(w, w, 64, 64, 64, 64, 1e-3)
    assert (g.q1, g.r1, g.p1) == (8, 9, 64)
    r = ref.RefPlan.create(DATA / "scope_table_v1.txt", w, w, 64, 64, 64, 64, 1e-3)
    dcrop = np.stack([ref.crop_centered(dj.astype(np.float64), 64, 64) for dj in d]).astype(np.float32)
    fs, bs = P.evaluate(torch.from_numpy(obj).cuda(), torch.from_numpy(probe).cuda(), offs,
                        torch.from_numpy(d).cuda(), plan=g, d_crop=torch.from_numpy(dcrop).cuda())
    o64, p64 = obj.astype(np.complex128), probe.astype(np.complex128)
    want_b = 0.0
    for j, (r0, c0) in enumerate(offs):
        ex = p64 * o64[r0:r0 + w, c0:c0 + w]
        want_b += np.sum((np.abs(r.apply(ex)) - dcrop[j]) ** 2)
    want_f = ref.objective_value(o64, p64, offs, d.astype(np.float64)) * len(offs)
    assert abs(bs - want_b) <= 1e-5 * want_b
    assert abs(fs - want_f) <= 1e-5 * want_f


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_crop_centered_bit_exact(ref, dtype):
    """crop_centered(RealField) (fft.cpp:206-232) is pure index work: bit-exact
    against the reference, batched, odd band offsets and mt = n/2."""
    rng = np.random.default_rng(40)
    for (n1, n2, mt1, mt2) in ((512, 512, 64, 64), (64, 128, 5, 17), (32, 32, 16, 16), (16, 8, 1, 4)):
        d = (np.abs(cnormal(rng, (3, n1, n2))) * 7).astype(dtype)
        got = P.crop_centered(torch.from_numpy(d).cuda(), mt1, mt2).cpu().numpy()
        assert got.dtype == dtype
        for b in range(3):
            want = ref.crop_centered(d[b].astype(np.float64), mt1, mt2).astype(dtype)
            assert np.array_equal(got[b], want), (n1, n2, mt1, mt2, b)
    with pytest.raises(ValueError):
        P.crop_centered(torch.zeros((8, 8), device="cuda"), 5, 1)


def test_concurrent_streams_and_threads_bit_identical():
    """B4: plans are immutable and every call takes its own stream-ordered
    scratch, so concurrent calls -- two host threads, each on its own CUDA
    stream, plus the host-buffer entry points from both threads -- give results
    bit-identical to the serial run."""
    import threading
    g = P.pft_plan_2d(1024, 1024, 40, 40, 32, 32, 1e-3)
    g2 = P.pft_plan_2d(256, 256, 32, 32, 32, 32, 1e-3)
    rng = np.random.default_rng(41)
    zs = [torch.from_numpy(cnormal(rng, (6, 1024, 1024), np.complex64)).cuda() for _ in range(2)]
    hs = [cnormal(rng, (5, 256, 256), np.complex64) for _ in range(2)]
    serial = [P.pft_adjoint_2d(g, P.pft_apply_2d(g, z)) for z in zs]
    serial_h = [P.pft_apply_2d(g2, h) for h in hs]
    torch.cuda.synchronize()
    out, out_h, errs = [None, None], [None, None], []

    def work(k):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(4):
                    out[k] = P.pft_adjoint_2d(g, P.pft_apply_2d(g, zs[k]))
                    out_h[k] = P.pft_apply_2d(g2, hs[k])
            s.synchronize()
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=work, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for k in range(2):
        assert torch.equal(out[k], serial[k])
        assert np.array_equal(out_h[k], serial_h[k])


def test_window_bounds_and_operand_checks():
    """Out-of-frame windows raise IndexError (std::out_of_range) instead of a
    device fault; in-place operands must be contiguous and share dtype/device."""
    frame = torch.zeros((100, 90), dtype=torch.complex64, device="cuda")
    patch = torch.ones((32, 32), dtype=torch.complex64, device="cuda")
    for off in ((69, 0), (0, 59), (-1, 0), (0, -3)):
        with pytest.raises(IndexError):
            P.set_window(frame, off, patch)
        with pytest.raises(IndexError):
            P.window_slice(frame, np.array([off]), 32, 32)
    P.set_window(frame, (68, 58), patch)  # the last in-frame corner is fine
    assert torch.count_nonzero(frame) == 32 * 32
    with pytest.raises(ValueError):
        P.set_window(frame, (0, 0), patch.to(torch.complex128))
    with pytest.raises(ValueError):
        P.set_window(frame.t(), (0, 0), patch)
    z = torch.ones((16, 16), dtype=torch.complex64, device="cuda")
    with pytest.raises(ValueError):
        P.pie_object_update(z, z.to(torch.complex128), z, 0.5)
    with pytest.raises(ValueError):
        P.epie_probe_update(z, z, z.to(torch.complex128), 0.5, True)
    d = torch.ones((2, 32, 32), device="cuda")
    with pytest.raises(IndexError):
        P.evaluate(frame, patch, np.array([[0, 0], [80, 0]]), d)
    with pytest.raises(ValueError):
        P.evaluate(frame, patch, np.array([[0, 0], [10, 0], [20, 0]]), d)


def test_evaluator_cfg5_full_size_chunk_invariance_and_sample(ref):
    """BASELINE configs[4] at full size (1600 positions of 512^2 complex64 on the
    4096^2 cfg4 object, band M = 128): the one-call evaluation equals the sum of
    four position ranges (summation order only), and a sample of positions
    matches the reference (objective_value / pft_apply_2d in double on the
    complex64 inputs) within complex64 rounding."""
    from paper_2408_03532_b200 import problems as PR
    prob = PR.make_problem("cfg4", seed=0)
    obj = prob.obj * (1 + 0.05 * torch.randn(prob.obj.shape, dtype=torch.complex64, device="cuda",
                                            generator=torch.Generator(device="cuda").manual_seed(3)))
    w, npos = prob.probe.shape[0], len(prob.offsets)
    assert npos == 1600 and w == 512
    plan = P.pft_plan_2d(w, w, 64, 64, 64, 64, 1e-3)
    dcrop = P.crop_centered(prob.d, 64, 64)
    fs, bs = P.evaluate(obj, prob.probe, prob.offsets, prob.d, (0, npos), plan, dcrop)
    parts = [P.evaluate(obj, prob.probe, prob.offsets, prob.d, (b, e), plan, dcrop)
             for b, e in ((0, 400), (400, 800), (800, 1200), (1200, 1600))]
    assert abs(fs - sum(p[0] for p in parts)) <= 1e-12 * fs
    assert abs(bs - sum(p[1] for p in parts)) <= 1e-12 * bs
    o64 = obj.cpu().numpy().astype(np.complex128)
    p64 = prob.probe.cpu().numpy().astype(np.complex128)
    d64 = prob.d.cpu().numpy().astype(np.float64)
    dc = dcrop.cpu().numpy().astype(np.float64)
    r = ref.RefPlan.create(DATA / "scope_table_v1.txt", w, w, 64, 64, 64, 64, 1e-3)
    for j in (0, 777, 1599):
        gf, gb = P.evaluate(obj, prob.probe, prob.offsets, prob.d, (j, j + 1), plan, dcrop)
        o = prob.offsets[j]
        want_f = ref.objective_value(o64, p64, [o], d64[j:j + 1])
        ex = p64 * o64[o[0]:o[0] + w, o[1]:o[1] + w]
        want_b = np.sum((np.abs(r.apply(ex)) - dc[j]) ** 2)
        assert abs(gf - want_f) <= 1e-4 * want_f, (j, gf, want_f)
        assert abs(gb - want_b) <= 1e-4 * want_b, (j, gb, want_b)


_PERSIST_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2408_03532_b200 as P
rng = np.random.default_rng(31)
out = {}
for w, n, blind, band in ((256, 400, True, 0), (256, 400, False, 0), (512, 700, True, 0), (256, 400, True, 1),
                         (512, 700, True, 1), (256, 400, False, 1)):
    obj = (rng.random((n, n)) * np.exp(1j * rng.random((n, n)))).astype(np.complex64)
    probe = np.exp(-((np.arange(w) - w / 2) ** 2)[:, None] / (w * w / 8.0)
                   - ((np.arange(w) - w / 2) ** 2)[None, :] / (w * w / 8.0)).astype(np.complex64)
    offs = np.array([[r, c] for r in (0, 37, n - w) for c in (0, 51, n - w)], np.int64)
    d = (np.abs(rng.standard_normal((len(offs), w, w))) * 30).astype(np.float32)
    cfg = P.SolverConfig(pft_sweeps=2 * band, fft_sweeps=2 * (1 - band), beta=0.5, gamma=0.05,
                         beta_pft=0.25 / w ** 2, gamma_pft=0.0125 / w ** 2, eps_pft=1e-3, blind=blind)
    r = P.hybrid_solve(d, offs, probe, obj, cfg)
    out[f"f{w}{int(blind)}{band}"] = r.frame
    out[f"p{w}{int(blind)}{band}"] = r.probe
np.savez(sys.argv[2], **out)
"""


def test_persistent_fft_sweep_bit_identical(tmp_path):
    """The persistent cooperative sweeps (epie_sweep.cuh full-FFT stage,
    band_sweep.cuh PFT-band stage) run the same arithmetic as the per-position
    kernel graphs: frames and probes after two sweeps are bit-identical
    (FFT stage 256^2 blind / non-blind and 512^2 blind; band stage 256^2 / 512^2
    blind, p = 32 / 64, q = 8, r = 9)."""
    import os
    import subprocess
    import sys
    from conftest import ROOT
    script = tmp_path / "persist.py"
    script.write_text(_PERSIST_SCRIPT)
    res = {}
    # PFTG_EVAL_BAND_OLD=12: the band stage on the streaming kernels, whose bodies the
    # persistent band sweep shares (the default band stage runs eval_band.cu's kernels
    # per position, see test_band_stage_axis_reordered_kernels)
    # PFTG_PERSIST=1: the persistent sweeps (the default is the per-position graph, whose
    # kernels are chained by programmatic dependent launch)
    for tag, extra in (("persist", {"PFTG_PERSIST": "1"}), ("graph", {"PFTG_NO_PERSIST": "1"})):
        env = {**os.environ, "PFTG_EVAL_BAND_OLD": "12", **extra}
        out = tmp_path / f"{tag}.npz"
        subprocess.run([sys.executable, str(script), str(ROOT), str(out)], env=env, check=True, timeout=600)
        res[tag] = np.load(out)
    for k in res["persist"].files:
        assert np.array_equal(res["persist"][k], res["graph"][k]), k


def test_band_stage_axis_reordered_kernels(tmp_path):
    """The default PFT-band stage of the q = 8, r = 9 complex64 plans runs the
    axis-reordered kernels of eval_band.cu (kb_cols: radix-8 column transforms
    with the residual and the adjoint gather in registers; kb_adj_rows: A-dagger
    on the band side, epilogue and fused forward per output row). Same operator
    sequence as the streaming kernels (PFTG_EVAL_BAND_OLD=12), different
    summation order: frames and probes after two blind band sweeps agree to
    complex64 rounding."""
    import os
    import subprocess
    import sys
    from conftest import ROOT
    script = tmp_path / "band.py"
    script.write_text(_PERSIST_SCRIPT)
    res = {}
    for tag, extra in (("new", {}), ("old", {"PFTG_EVAL_BAND_OLD": "12"})):
        env = {**os.environ, **extra}
        out = tmp_path / f"{tag}.npz"
        subprocess.run([sys.executable, str(script), str(ROOT), str(out)], env=env, check=True, timeout=600)
        res[tag] = np.load(out)
    for k in res["new"].files:
        a, b = res["new"][k], res["old"][k]
        err = np.linalg.norm(a - b) / np.linalg.norm(b)
        if k.endswith("1"):  # band-stage cases
            assert err <= 2e-5, (k, err)
        else:
            assert np.array_equal(a, b), k


def test_pdl_chained_positions_bit_identical(tmp_path):
    """The kernels of an ePIE position are chained by programmatic dependent launch
    (each waits, then releases its successor, whose table loads and operand prefetch
    run ahead of its own wait). Hazard check: frames and probes after two sweeps are
    bit-identical with plain serialized launches (PFTG_EB_NO_PDL / PFTG_FFT_NO_PDL),
    for the full-FFT stage (256^2 blind / non-blind, 512^2) and the band stage
    (p = 32 and p = 64 plans)."""
    import os
    import subprocess
    import sys
    from conftest import ROOT
    script = tmp_path / "pdl.py"
    script.write_text(_PERSIST_SCRIPT)
    res = {}
    for tag, extra in (("pdl", {}), ("plain", {"PFTG_EB_NO_PDL": "1", "PFTG_FFT_NO_PDL": "1"})):
        env = {**os.environ, **extra}
        out = tmp_path / f"{tag}.npz"
        subprocess.run([sys.executable, str(script), str(ROOT), str(out)], env=env, check=True, timeout=600)
        res[tag] = np.load(out)
    for k in res["pdl"].files:
        assert np.array_equal(res["pdl"][k], res["plain"][k]), k
