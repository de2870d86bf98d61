"""GPU parity against the committed golden fixtures (produced by the reference
itself, tests/golden/make_golden.py) and the numpy oracle port -- these need
neither /root/reference nor oracle/_ref on the GPU box."""
import numpy as np
import pytest

from conftest import DATA, GOLDEN, cnormal, rel_l2

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2408_03532_b200")
from oracle import pft_oracle as O  # noqa: E402


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_pft_small_golden_c128():
    g = np.load(GOLDEN / "pft_small.npz")
    pl = P.pft_plan_2d(64, 64, 8, 8, 8, 8, 1e-7)
    assert rel_l2(P.pft_apply_2d(pl, cuda(g["z"])).cpu().numpy(), g["band"]) <= 1e-10
    assert rel_l2(P.pft_adjoint_2d(pl, cuda(g["y"])).cpu().numpy(), g["adj"]) <= 1e-10


def test_pft_rect_golden_c128():
    g = np.load(GOLDEN / "pft_rect.npz")
    pl = P.pft_plan_2d(128, 64, 4, 8, 16, 8, 1e-3)
    assert rel_l2(P.pft_apply_2d(pl, cuda(g["z"])).cpu().numpy(), g["band"]) <= 1e-10
    assert rel_l2(P.pft_adjoint_2d(pl, cuda(g["y"])).cpu().numpy(), g["adj"]) <= 1e-10


def test_pft_cfg1_literal_golden_c128():
    """BASELINE configs[0]: 512^2 complex128, p=16, q=32, r=12, M=128 (rel L2 <= 1e-10)."""
    g = np.load(GOLDEN / "pft_cfg1_literal.npz")
    pl = P.pft_plan_2d(512, 512, 64, 64, 16, 16, 1.0, P.ScopeTable.load(DATA / "scope_table_xi4_r12.txt"))
    z = cnormal(np.random.default_rng(int(g["seed"])), (512, 512))
    assert rel_l2(P.pft_apply_2d(pl, cuda(z)).cpu().numpy(), g["band"]) <= 1e-10
    adj = P.pft_adjoint_2d(pl, cuda(g["band"])).cpu().numpy()
    assert rel_l2(adj[::7, ::13], g["adj_sample"]) <= 1e-10


def test_cfg1_fft_crop_deviation_reported():
    """The literal cfg1 plan is outside the PFT accuracy domain (xi = 4): the band
    is far from the exact FFT crop -- identically for the GPU and the reference."""
    g = np.load(GOLDEN / "pft_cfg1_literal.npz")
    z = cnormal(np.random.default_rng(int(g["seed"])), (512, 512))
    crop = O.crop_centered(np.fft.fft2(z), 64, 64)
    pl = P.pft_plan_2d(512, 512, 64, 64, 16, 16, 1.0, P.ScopeTable.load(DATA / "scope_table_xi4_r12.txt"))
    gpu = P.pft_apply_2d(pl, cuda(z)).cpu().numpy()
    assert abs(rel_l2(gpu, crop) - rel_l2(g["band"], crop)) <= 1e-9


def test_solver_tiny_golden_c128():
    g = np.load(GOLDEN / "solver_tiny.npz")
    cfg = g["hybrid_cfg"]
    res = P.hybrid_solve(g["d"], g["offs"], g["probe"] * 0.9, g["init"],
                         P.SolverConfig(pft_sweeps=int(cfg[0]), fft_sweeps=int(cfg[1]), beta=cfg[2],
                                        gamma=cfg[3], beta_pft=cfg[4], gamma_pft=cfg[5], eps_pft=cfg[6],
                                        blind=True),
                         dtype=np.complex128)
    assert rel_l2(res.frame, g["hybrid_frame"]) <= 1e-9
    assert rel_l2(res.probe, g["hybrid_probe"]) <= 1e-9
    assert np.allclose(res.objective, g["hybrid_objective"], rtol=1e-8)


def test_blocks_golden():
    g = np.load(GOLDEN / "solver_tiny.npz")
    pm = P.project_modulus(cuda(g["x"]), cuda(g["dn"])).cpu().numpy()
    assert rel_l2(pm, g["project_modulus"]) <= 1e-12
    pl = P.pft_plan_2d(64, 64, 8, 8, 8, 8, 1e-3)
    br = P.band_residual(pl, cuda(g["x"]), cuda(g["dcrop"])).cpu().numpy()
    assert rel_l2(br, g["band_residual"]) <= 1e-10
    phi = P.objective_value(cuda(g["init"]), cuda(g["probe"]), g["offs"], cuda(g["d"]))
    assert abs(phi - g["phi0"]) <= 1e-10 * g["phi0"]


@pytest.mark.parametrize("shape", [(256, 256, 32, 32, 32, 32, 1e-3), (512, 512, 64, 64, 64, 64, 1e-3)])
def test_port_parity_c64(shape):
    """complex64 GPU vs the numpy port in double on the rounded inputs: rel L2 <= 1e-5
    (scope-1 plans of BASELINE configs[2..4])."""
    n1, n2, mt1, mt2, p1, p2, eps = shape
    pl = P.pft_plan_2d(*shape)
    po = O.plan_2d(*shape, O.load_scope_table(DATA / "scope_table_v1.txt"))
    rng = np.random.default_rng(9)
    z = cnormal(rng, (3, n1, n2), np.complex64)
    band = P.pft_apply_2d(pl, cuda(z)).cpu().numpy()
    back = P.pft_adjoint_2d(pl, cuda(band)).cpu().numpy()
    for b in range(3):
        want = O.pft_apply_2d(po, z[b].astype(np.complex128))
        assert rel_l2(band[b], want) <= 1e-5
        assert rel_l2(back[b], O.pft_adjoint_2d(po, band[b].astype(np.complex128))) <= 1e-5
