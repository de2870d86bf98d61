"""B1 drop-in demonstration: the reference library built VERBATIM from its own
sources (oracle/Makefile) with the C++ façade paper_2408_03532_b200/facade/
pft_gpu.cpp providing ptycho::pft::pft_apply_2d / pft_adjoint_2d and
ptycho::fast_fft2 / fast_ifft2 over libpftg. The reference's unmodified
solver.cpp (project_modulus, band_residual, hybrid_solve) then runs on the GPU
transforms; its results must match the all-CPU reference build."""
import numpy as np
import pytest

from conftest import DATA, cnormal, rel_l2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fac(ref):
    if not ref.FACADE_PATH.exists():
        pytest.skip("façade build missing (make -C oracle)")
    return ref


def test_facade_pft_and_fft_match_reference(fac):
    rng = np.random.default_rng(60)
    z = cnormal(rng, (512, 512))
    y = cnormal(rng, (128, 128))
    cpu = fac.RefPlan.create(DATA / "scope_table_v1.txt", 512, 512, 64, 64, 64, 64, 1e-7)
    with fac.facade():
        gpu = fac.RefPlan.create(DATA / "scope_table_v1.txt", 512, 512, 64, 64, 64, 64, 1e-7)
        assert rel_l2(gpu.apply(z), cpu.apply(z)) <= 1e-10
        assert rel_l2(gpu.adjoint(y), cpu.adjoint(y)) <= 1e-10
        f_gpu, fi_gpu = fac.fast_fft2(z), fac.fast_ifft2(z)
        with pytest.raises(ValueError):
            gpu.apply(z[:256])  # invalid_argument from the façade, as from pft.cpp:122-123
    assert rel_l2(f_gpu, fac.fast_fft2(z)) <= 1e-13
    assert rel_l2(fi_gpu, fac.fast_ifft2(z)) <= 1e-13


@pytest.mark.parametrize("blind", [False, True])
def test_verbatim_hybrid_solve_on_gpu_transforms(fac, blind):
    """hybrid_solve (solver.cpp:173-302, compiled verbatim) over the façade:
    band stage (band_residual -> GPU pft_apply_2d / pft_adjoint_2d) and full-FFT
    stage (project_modulus -> GPU fast_fft2 / fast_ifft2), object + probe after
    2 + 2 sweeps and the per-sweep objective equal the all-CPU reference to 1e-9."""
    rng = np.random.default_rng(61)
    n, w = 160, 64
    obj = (0.5 + 0.5 * rng.random((n, n))) * np.exp(1j * rng.uniform(-1, 1, (n, n)))
    yy, xx = np.mgrid[0:w, 0:w] - (w - 1) / 2
    probe = np.exp(-(xx ** 2 + yy ** 2) / (2 * 13.0 ** 2)) * np.exp(1j * 0.3 * (xx ** 2 + yy ** 2) / w ** 2)
    pos = np.linspace(0, n - w, 3).round().astype(int)
    offs = np.array([[r, c] for r in pos for c in pos], np.int64)
    d = fac.simulate(obj, probe, offs)
    init = np.exp(1j * 0.1 * rng.standard_normal((n, n))) * 0.8
    kw = dict(pft_sweeps=2, fft_sweeps=2, beta=0.5, gamma=0.05, beta_pft=0.25 / w ** 2,
              gamma_pft=0.0125 / w ** 2, eps_pft=1e-3, blind=blind,
              table_path=DATA / "scope_table_v1.txt")
    f_cpu, p_cpu, o_cpu, _, fl_cpu = fac.hybrid_solve(init, probe * 0.9, offs, d, **kw)
    with fac.facade():
        f_gpu, p_gpu, o_gpu, _, fl_gpu = fac.hybrid_solve(init, probe * 0.9, offs, d, **kw)
    assert fl_cpu == fl_gpu == 0 and len(o_gpu) == 4
    assert rel_l2(f_gpu, f_cpu) <= 1e-9
    assert rel_l2(p_gpu, p_cpu) <= 1e-9
    assert np.allclose(o_gpu, o_cpu, rtol=1e-9)


def test_facade_pft_apply_1d_matches_reference(fac):
    rng = np.random.default_rng(61)
    z = rng.standard_normal(4096) + 1j * rng.standard_normal(4096)
    cpu = fac.RefPlan1D.create(DATA / "scope_table_v1.txt", 4096, 128, 128, 1e-3)
    want = cpu.apply(z)
    with fac.facade():
        gpu = fac.RefPlan1D.create(DATA / "scope_table_v1.txt", 4096, 128, 128, 1e-3)
        got = gpu.apply(z)
    assert rel_l2(got, want) <= 1e-10
