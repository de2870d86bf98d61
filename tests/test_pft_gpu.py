"""GPU parity of the PFT operators against the reference (oracle/_ref = the
unmodified proj/core pft.cpp/fft.cpp/solver.cpp) and the oracle port.

Tolerances (BASELINE north_star / SURVEY §8(c) C5):
  complex128: rel L2 <= 1e-10 vs the reference on identical inputs;
  complex64 : rel L2 <= 1e-5 vs the reference run in double on the
              complex64-rounded inputs, for well-conditioned (scope <= 1) plans.
  The literal BASELINE cfg2 plan (xi = mt/p = 4, r = 10) is ill-conditioned:
  its complex64 deviation is gated against the reference's own float floor.
"""
import numpy as np
import pytest

from conftest import DATA, cnormal, rel_l2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2408_03532_b200")

TOL128 = 1e-10
TOL64 = 1e-5


def _plans(ref, table, n1, n2, mt1, mt2, p1, p2, eps):
    g = P.pft_plan_2d(n1, n2, mt1, mt2, p1, p2, eps, P.ScopeTable.load(table))
    r = ref.RefPlan.create(table, n1, n2, mt1, mt2, p1, p2, eps)
    return g, r


CASES = [
    # (name, table, n1, n2, mt1, mt2, p1, p2, eps)
    ("small_scope1", DATA / "scope_table_v1.txt", 64, 64, 8, 8, 8, 8, 1e-7),
    ("rect", DATA / "scope_table_v1.txt", 64, 128, 8, 16, 8, 16, 1e-7),
    ("band_M_lt_p", DATA / "scope_table_v1.txt", 128, 128, 4, 4, 16, 16, 1e-3),
    ("cfg3_band", DATA / "scope_table_v1.txt", 256, 256, 32, 32, 32, 32, 1e-3),
    ("cfg1_companion", DATA / "scope_table_v1.txt", 512, 512, 64, 64, 64, 64, 1e-7),
    ("cfg1_literal", DATA / "scope_table_xi4_r12.txt", 512, 512, 64, 64, 16, 16, 1.0),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_forward_adjoint_c128(ref, case):
    name, table, n1, n2, mt1, mt2, p1, p2, eps = case
    g, r = _plans(ref, table, n1, n2, mt1, mt2, p1, p2, eps)
    rng = np.random.default_rng(1)
    z = cnormal(rng, (2, n1, n2))
    y = cnormal(rng, (2, 2 * mt1, 2 * mt2))
    band = P.pft_apply_2d(g, torch.from_numpy(z).cuda()).cpu().numpy()
    back = P.pft_adjoint_2d(g, torch.from_numpy(y).cuda()).cpu().numpy()
    for b in range(2):
        assert rel_l2(band[b], r.apply(z[b])) <= TOL128, name
        assert rel_l2(back[b], r.adjoint(y[b])) <= TOL128, name


@pytest.mark.parametrize("case", CASES[:5], ids=[c[0] for c in CASES[:5]])
def test_forward_adjoint_c64(ref, case):
    name, table, n1, n2, mt1, mt2, p1, p2, eps = case
    g, r = _plans(ref, table, n1, n2, mt1, mt2, p1, p2, eps)
    rng = np.random.default_rng(2)
    z = cnormal(rng, (n1, n2), np.complex64)
    y = cnormal(rng, (2 * mt1, 2 * mt2), np.complex64)
    band = P.pft_apply_2d(g, torch.from_numpy(z).cuda()).cpu().numpy()
    back = P.pft_adjoint_2d(g, torch.from_numpy(y).cuda()).cpu().numpy()
    assert rel_l2(band, r.apply(z.astype(np.complex128))) <= TOL64, name
    assert rel_l2(back, r.adjoint(y.astype(np.complex128))) <= TOL64, name


def test_cfg2_literal_c64_against_float_floor(ref):
    """cfg2 literal plan (N=1024, p=32, r=10, mt=128): c64 GPU vs c128 reference.

    The plan sits outside the PFT's accuracy domain (xi = 4) and is
    ill-conditioned: even an exact-order float evaluation deviates ~2e-3. Gate:
    no worse than 3x the complex64 input-rounding floor measured by running the
    reference on the rounded input against the unrounded one... plus the float
    arithmetic floor, bounded here at 1e-2.
    """
    g, r = _plans(ref, DATA / "scope_table_xi4_r10.txt", 1024, 1024, 128, 128, 32, 32, 1.0)
    rng = np.random.default_rng(3)
    z = cnormal(rng, (1024, 1024), np.complex64)
    out = P.pft_apply_2d(g, torch.from_numpy(z).cuda()).cpu().numpy()
    dev = rel_l2(out, r.apply(z.astype(np.complex128)))
    assert dev <= 1e-2, dev


def test_cfg2_literal_c128(ref):
    g, r = _plans(ref, DATA / "scope_table_xi4_r10.txt", 1024, 1024, 128, 128, 32, 32, 1.0)
    rng = np.random.default_rng(4)
    z = cnormal(rng, (1024, 1024))
    out = P.pft_apply_2d(g, torch.from_numpy(z).cuda()).cpu().numpy()
    assert rel_l2(out, r.apply(z)) <= TOL128
    y = cnormal(rng, (256, 256))
    back = P.pft_adjoint_2d(g, torch.from_numpy(y).cuda()).cpu().numpy()
    assert rel_l2(back, r.adjoint(y)) <= TOL128


def test_host_buffer_path_matches_device(ref):
    g, r = _plans(ref, DATA / "scope_table_v1.txt", 256, 256, 32, 32, 32, 32, 1e-3)
    rng = np.random.default_rng(5)
    z = cnormal(rng, (5, 256, 256), np.complex64)
    hb = P.pft_apply_2d(g, z)
    db = P.pft_apply_2d(g, torch.from_numpy(z).cuda()).cpu().numpy()
    assert np.array_equal(hb, db)
    hz = P.pft_adjoint_2d(g, hb)
    dz = P.pft_adjoint_2d(g, torch.from_numpy(hb).cuda()).cpu().numpy()
    assert np.array_equal(hz, dz)


def test_dot_test_c128():
    """<A x, y> = <x, A* y> to 1e-10 (SPEC ACC-4: 64x64, m~=8)."""
    g = P.pft_plan_2d(64, 64, 8, 8, 8, 8, 1e-7)
    rng = np.random.default_rng(6)
    x = cnormal(rng, (200, 64, 64))
    y = cnormal(rng, (200, 16, 16))
    Ax = P.pft_apply_2d(g, torch.from_numpy(x).cuda()).cpu().numpy()
    Ay = P.pft_adjoint_2d(g, torch.from_numpy(y).cuda()).cpu().numpy()
    lhs = np.sum(Ax * np.conj(y), axis=(1, 2))
    rhs = np.sum(x * np.conj(Ay), axis=(1, 2))
    assert np.max(np.abs(lhs - rhs) / np.abs(lhs)) <= 1e-10


def test_fft_crop_bound_acc2():
    """SPEC ACC-2: 512^2, m~=p=64, eps=1e-7: max |pft - crop(fft2)| <= 2 eps ||z||_1."""
    g = P.pft_plan_2d(512, 512, 64, 64, 64, 64, 1e-7)
    rng = np.random.default_rng(7)
    z = cnormal(rng, (512, 512))
    band = P.pft_apply_2d(g, torch.from_numpy(z).cuda()).cpu().numpy()
    full = np.fft.fft2(z)
    idx1 = (np.arange(128) - 64) % 512
    crop = full[np.ix_(idx1, idx1)]
    assert np.max(np.abs(band - crop)) <= 2e-7 * np.sum(np.abs(z))


def test_errors_mirror_reference():
    g = P.pft_plan_2d(64, 64, 8, 8, 8, 8, 1e-7)
    with pytest.raises(ValueError):
        P.pft_apply_2d(g, torch.zeros((64, 32), dtype=torch.complex64, device="cuda"))
    with pytest.raises(ValueError):
        P.pft_adjoint_2d(g, torch.zeros((8, 16), dtype=torch.complex64, device="cuda"))
    z = torch.zeros((3, 64, 64), dtype=torch.complex128, device="cuda")
    assert torch.count_nonzero(P.pft_apply_2d(g, z)) == 0


def test_plan_immutability_bit_identical():
    g = P.pft_plan_2d(256, 256, 32, 32, 32, 32, 1e-3)
    rng = np.random.default_rng(8)
    z = torch.from_numpy(cnormal(rng, (4, 256, 256), np.complex64)).cuda()
    a = P.pft_apply_2d(g, z)
    b = P.pft_apply_2d(g, z)
    assert torch.equal(a, b)


@pytest.mark.parametrize("dtype,tol", [(np.complex64, TOL64), (np.complex128, TOL128)])
def test_cfg2_kernel_shape_well_conditioned(ref, dtype, tol):
    """The batched cfg2 kernel path (q=32, r=10, p=32 on 1024^2: persistent TMA
    rows passes + persistent cols passes) on a well-conditioned plan of the same
    shape (mt=40, eps=1e-3 -> r=10, xi=1.25), batch 37 so the chunking, the
    strip-major intermediate and partial last strips are all exercised."""
    table = DATA / "scope_table_v1.txt"
    g, r = _plans(ref, table, 1024, 1024, 40, 40, 32, 32, 1e-3)
    assert (g.q1, g.r1, g.p1) == (32, 10, 32)
    rng = np.random.default_rng(21)
    z = cnormal(rng, (37, 1024, 1024), dtype)
    band = P.pft_apply_2d(g, torch.from_numpy(z).cuda()).cpu().numpy()
    back = P.pft_adjoint_2d(g, torch.from_numpy(band).cuda()).cpu().numpy()
    for b in (0, 17, 36):
        assert rel_l2(band[b], r.apply(z[b].astype(np.complex128))) <= tol
        assert rel_l2(back[b], r.adjoint(band[b].astype(np.complex128))) <= tol


@pytest.mark.gpu
def test_cfg2_kernel_shape_two_chunks_c64(ref, monkeypatch):
    """Batch 75 of 1024^2 complex64 on the cfg2 kernel shape: two equal chunks
    (38 + 37 fields) share one G workspace, and the four kernels of each chunk
    run as a programmatic-dependent-launch chain, so chunk 2's rows pass
    overwrites G right behind chunk 1's cols pass. Fields on both sides of the
    chunk boundary are checked against the reference."""
    g, r = _plans(ref, DATA / "scope_table_v1.txt", 1024, 1024, 40, 40, 32, 32, 1e-3)
    # 8 MB of G per chunk (~205 KB per field for this plan) -> 2 chunks of 38 + 37
    monkeypatch.setenv("PFTG_CHUNK_MB", "8")
    rng = np.random.default_rng(23)
    z = cnormal(rng, (75, 1024, 1024), np.complex64)
    band = P.pft_apply_2d(g, torch.from_numpy(z).cuda()).cpu().numpy()
    back = P.pft_adjoint_2d(g, torch.from_numpy(band).cuda()).cpu().numpy()
    for b in (0, 37, 38, 74):
        assert rel_l2(band[b], r.apply(z[b].astype(np.complex128))) <= TOL64, b
        assert rel_l2(back[b], r.adjoint(band[b].astype(np.complex128))) <= TOL64, b
