"""GPU parity of the steps either side of the hot path:
F1 measurement simulator (simulate / add_poisson_noise / build_cropped,
simulate.cpp:48-89) and F2 per-sweep metrics (metrics.cpp:60-143,
fill_metrics solver.cpp:141-160), against the reference (oracle/_ref)."""
import numpy as np
import pytest

from conftest import cnormal, rel_l2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2408_03532_b200")


@pytest.mark.parametrize("dtype,tol", [(np.complex128, 1e-13), (np.complex64, 1e-6)])
@pytest.mark.parametrize("w", [64, 256, 512])
def test_simulate_matches_reference(ref, dtype, tol, w):
    rng = np.random.default_rng(70 + w)
    n = w + 70
    frame = cnormal(rng, (n, n), dtype)
    probe = cnormal(rng, (w, w), dtype)
    offs = np.array([[0, 0], [3, 7], [70, 70], [35, 1], [69, 68]], np.int64)
    d = P.simulate(torch.from_numpy(frame).cuda(), torch.from_numpy(probe).cuda(), offs).cpu().numpy()
    want = ref.simulate(frame.astype(np.complex128), probe.astype(np.complex128), offs)
    assert d.dtype == (np.float64 if dtype == np.complex128 else np.float32)
    for j in range(len(offs)):
        assert rel_l2(d[j], want[j]) <= tol, j
    dc = P.build_cropped(torch.from_numpy(d).cuda(), w // 8, w // 8).cpu().numpy()
    assert np.array_equal(dc[2], ref.crop_centered(d[2].astype(np.float64), w // 8, w // 8).astype(d.dtype))
    with pytest.raises(IndexError):
        P.simulate(torch.from_numpy(frame).cuda(), torch.from_numpy(probe).cuda(), np.array([[71, 0]]))


def test_poisson_noise_law_and_reproducibility(ref):
    """add_poisson_noise: d <- sqrt(Poisson(s d^2)/s). Per lambda group (both
    samplers: inversion below 10, PTRS above) the counts' mean and variance
    match lambda within 6 standard errors, for our stream and for the
    reference's own libstdc++ stream on the same input; zeros stay zero; the
    same seed reproduces bit for bit, another seed does not."""
    lams = np.array([0.0, 0.3, 2.5, 9.9, 10.0, 37.0, 1000.0, 2.5e5])
    per = 1 << 16
    scale = 4.0
    d0 = np.repeat(np.sqrt(lams / scale), per).astype(np.float64)
    dt = torch.from_numpy(d0.copy()).cuda()
    P.add_poisson_noise(dt, scale, 1234)
    k = (dt.cpu().numpy() ** 2 * scale).round().reshape(len(lams), per)
    dref = ref.add_poisson_noise(d0.reshape(len(lams), per, 1), scale, 1234)
    kref = (dref.reshape(len(lams), per) ** 2 * scale).round()
    for i, lam in enumerate(lams):
        for kk in (k[i], kref[i]):
            if lam == 0:
                assert np.all(kk == 0)
                continue
            se_mean = np.sqrt(lam / per)
            assert abs(kk.mean() - lam) <= 6 * se_mean, (lam, kk.mean())
            # var of the sample variance of a Poisson: (lam + 2 lam^2) / per (approx.)
            se_var = np.sqrt((lam + 2 * lam * lam) / per)
            assert abs(kk.var() - lam) <= 6 * se_var, (lam, kk.var())
    again = torch.from_numpy(d0.copy()).cuda()
    P.add_poisson_noise(again, scale, 1234)
    assert torch.equal(again, dt)
    other = torch.from_numpy(d0.copy()).cuda()
    P.add_poisson_noise(other, scale, 1235)
    assert not torch.equal(other, dt)
    f32 = torch.from_numpy(d0.astype(np.float32)).cuda()
    P.add_poisson_noise(f32, scale, 1234)
    assert torch.isfinite(f32).all()
    with pytest.raises(ValueError):
        P.add_poisson_noise(f32, 0.0, 1)


@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
def test_fill_metrics_match_reference(ref, dtype):
    """The per-sweep metrics row: relative errors (plain, aligned, magnitude,
    phase), SSIM and PSNR of magnitude and phase, on an object region viewed
    inside a larger frame (row stride honoured), vs the reference's
    metrics.cpp on the same values."""
    rng = np.random.default_rng(80)
    truth = (0.5 + 0.5 * rng.random((140, 150))) * np.exp(1j * rng.uniform(-3, 3, (140, 150)))
    recon = truth * np.exp(1j * 0.7) + 0.05 * cnormal(rng, truth.shape)
    recon[3, 4] = 0  # arg(0) = 0 (field.cpp:84)
    frame = np.zeros((160, 170), np.complex128)
    frame[5:145, 9:159] = recon
    tr, fr_ = truth.astype(dtype), frame.astype(dtype)
    want = ref.fill_metrics(fr_[5:145, 9:159].astype(np.complex128), tr.astype(np.complex128))
    ft = torch.from_numpy(fr_).cuda()
    got = P.fill_metrics(ft[5:145, 9:159], torch.from_numpy(tr).cuda())
    vals = [got.rel_err, got.rel_err_aligned, got.rel_err_mag, got.rel_err_phase, got.ssim_mag, got.ssim_phase,
            got.psnr_mag, got.psnr_phase]
    for name, g, w in zip(P.metrics.FIELDS, vals, want):
        assert abs(g - w) <= 1e-11 * max(1.0, abs(w)), (name, g, w)
    assert got.rel_err_aligned < got.rel_err  # the global phase 0.7 is divided out
    same = P.fill_metrics(torch.from_numpy(tr).cuda(), torch.from_numpy(tr).cuda())
    assert same.rel_err == 0 and same.rel_err_aligned <= 1e-7 and same.psnr_mag == float("inf")
    assert abs(same.ssim_mag - 1) <= 1e-12
    with pytest.raises(ValueError):
        P.fill_metrics(torch.zeros((8, 8), dtype=torch.complex128, device="cuda"),
                       torch.zeros((8, 8), dtype=torch.complex128, device="cuda"))


def test_solver_metrics_trace_matches_reference(ref):
    """Per-sweep metrics of a device-resident solve (Solver.metrics after each
    sweep) equal the reference's fill_metrics of the same frame."""
    rng = np.random.default_rng(81)
    n, w = 128, 64
    truth = (0.5 + 0.5 * rng.random((n, n))) * np.exp(1j * rng.uniform(-1, 1, (n, n)))
    yy, xx = np.mgrid[0:w, 0:w] - (w - 1) / 2
    probe = np.exp(-(xx ** 2 + yy ** 2) / (2 * 13.0 ** 2)).astype(np.complex128)
    pos = np.linspace(0, n - w, 3).round().astype(int)
    offs = np.array([[r, c] for r in pos for c in pos], np.int64)
    d = ref.simulate(truth, probe, offs)
    init = np.ones((n, n), np.complex128) * 0.8
    cfg = P.SolverConfig(pft_sweeps=1, fft_sweeps=2, beta=0.5, gamma=0.05, beta_pft=0.25 / w ** 2,
                         gamma_pft=0.0125 / w ** 2, eps_pft=1e-3, blind=True)
    s = P.Solver(d, offs, probe, init, cfg, dtype=np.complex128)
    tt = torch.from_numpy(truth).cuda()
    for _ in range(3):
        s.run(1)
        m = s.metrics(tt)
        want = ref.fill_metrics(s.result().frame, truth)
        assert abs(m.rel_err_aligned - want[1]) <= 1e-11 * want[1]
        assert abs(m.ssim_phase - want[5]) <= 1e-11
