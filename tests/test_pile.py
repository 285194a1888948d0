"""configs[4] cube pile: host geometry, spatial-hash detection, face-side
nodalization (CPU), and the GPU pipeline (device augmentation + V-FPI solve)
stepped in lockstep with the CPU oracle (``-m gpu``)."""

import numpy as np
import pytest

from oracle import pile_host as H
from oracle import vfpi_oracle as O
from oracle.pile_host import contact_frames
from paper_2201_09212_b200.pile import CubePile, surface_triangles
from paper_2201_09212_b200.scenes import FemCube


def small_pile(**kw):
    args = dict(nx_cubes=2, ny_cubes=1, layers=2, nodes=4, gap=0.0, jitter=0.00005, seed=5, dt=5e-4)
    args.update(kw)
    return CubePile(**args)


def test_surface_is_closed_and_outward():
    cube = FemCube(nx=4)
    f = surface_triangles(4, cube.X)
    assert f.shape[0] == 6 * 3 * 3 * 2  # 6 faces x 9 quads x 2 triangles
    # closed surface: every edge shared by exactly two triangles
    e = np.sort(np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]]), axis=1)
    _, cnt = np.unique(e, axis=0, return_counts=True)
    assert (cnt == 2).all()
    # outward: the divergence theorem gives the (positive) volume
    P = cube.X[f]
    vol = np.einsum("ij,ij->i", P[:, 0], np.cross(P[:, 1], P[:, 2])).sum() / 6.0
    assert vol == pytest.approx(0.1 ** 3, rel=1e-12)


def test_contact_frames_match_scalar_frame():
    from paper_2201_09212_b200.contacts import contact_frame

    n = np.random.default_rng(0).standard_normal((50, 3))
    F = contact_frames(n)
    for k in range(50):
        assert np.allclose(F[k], contact_frame(n[k]), atol=1e-15)


def test_detection_and_nodalize_invariants():
    pile = small_pile()
    ground, face = H.detect(pile)
    assert ground.size and face["node"].size
    # node-to-face contacts couple different cubes, barycentric weights are a partition of unity
    assert (pile.node_cube[face["node"]] > pile.node_cube[face["tri"][:, 0]]).all()
    assert (face["w"] >= 0).all() and np.allclose(face["w"].sum(axis=1), 1.0)
    assert np.allclose(np.linalg.norm(face["normal"], axis=1), 1.0)
    assert np.unique(face["node"]).size == face["node"].size  # one face contact per node
    pc = H.nodalize(pile, ground, face)
    n_o = pile.n
    # plane contacts first: S contacts on the nodes' own slots
    assert (pc.col_j[: pc.n_ground] == -1).all() and (pc.col_i[: pc.n_ground] == 3 * ground).all()
    # face sides are virtual nodes; a node's second contact is an identity virtual node
    assert (pc.col_j[pc.n_ground:] >= n_o).all()
    both = np.intersect1d(ground, face["node"])
    assert both.size and (pc.col_i[pc.n_ground:] >= n_o).sum() == both.size
    cols = np.concatenate([pc.col_i, pc.col_j[pc.col_j >= 0]])
    assert np.unique(cols).size == cols.size  # diagonalization: one contact per node column
    # J_v rows: 9 stored entries per block (explicit zeros kept), each row sums to 1
    jv = pc.jv
    assert jv.shape == (3 * pc.n_virtual, n_o)
    assert np.allclose(np.asarray(jv.sum(axis=1)).ravel(), 1.0)
    assert (jv.data == 0).sum() == 2 * (jv.data != 0).sum()
    assert (pc.phi <= 0).all()


def _oracle_step(pile, prev, max_iters):
    pc = H.contacts(pile)
    b_o = H.rhs(pile)
    p, i, x, b = O.augment(pile.n, pile.a_indptr, pile.a_indices, pile.a_data, b_o, pc.jv, pile.k_v)
    s = O.System(pile.n + pc.jv.shape[0], p, i, x, b, pc.col_i, pc.col_j, pc.frames, pc.mu, pc.mu, pc.phi)
    warm = H.warm(pile, prev, pc)
    v, lam, rep = O.solve(s, O.Config(residual_tol=1e-8, max_iters=max_iters), warm)
    return pc, b_o, (p, i, x), warm, v, lam, rep


def test_oracle_pile_steps_touch_and_push():
    pile = small_pile()
    prev = None
    for _ in range(3):
        pc, _, _, _, v, lam, rep = _oracle_step(pile, prev, 100)
        assert pc.n_face > 0 and (lam[:, 0] >= 0).all()
        H.advance(pile, v)
        prev = v


@pytest.mark.gpu
def test_gpu_pile_lockstep_with_oracle():
    """Six steps: device augmentation bit-equal to the reference expression,
    GPU solve bit-equal to the oracle (plain strict V-FPI), same iterations."""
    from paper_2201_09212_b200.solver import SolverConfig, solve_packed

    pile = small_pile()
    prev = None
    for step in range(6):
        pc, b_o, (p, i, x), warm, vo, lo, ro = _oracle_step(pile, prev, 200)
        from paper_2201_09212_b200.augment import augment_arrays

        ps_p, ps_i, ps_x = augment_arrays(pile.n, pile.a_indptr, pile.a_indices, pile.a_data, pc.jv, pile.k_v)
        ps = H.system(pile, pc, b_o)
        assert np.array_equal(ps_p, p) and np.array_equal(ps_i, i) and np.array_equal(ps_x, x)
        assert np.array_equal(ps.indptr, p) and np.array_equal(ps.indices, i) and np.array_equal(ps.data, x)
        v, lam, rep = solve_packed(ps, SolverConfig(residual_tol=1e-8, max_iters=200), warm)
        assert rep.iterations == ro.iterations, step
        assert np.array_equal(v, vo), (step, float(np.abs(v - vo).max()))
        assert np.array_equal(lam, lo), step
        H.advance(pile, v)
        prev = v


@pytest.mark.gpu
def test_gpu_pile_stepper_matches_host_pipeline():
    """The device step pipeline (b, augmentation, warm start, solve,
    integration on the GPU) against the host pipeline driven by the oracle:
    same contacts and iterations every step, states bit-equal."""
    from paper_2201_09212_b200.pile import PileStepper
    from paper_2201_09212_b200.solver import SolverConfig

    host = small_pile()
    dev = PileStepper(small_pile())
    prev = None
    for step in range(6):
        pc, _, _, _, vo, lo, ro = _oracle_step(host, prev, 200)
        st = dev.step(SolverConfig(residual_tol=1e-8, max_iters=200))
        assert st["n_c"] == pc.n_c and st["n_face"] == pc.n_face
        assert st["iterations"] == ro.iterations, step
        H.advance(host, vo)
        prev = vo
        assert np.array_equal(dev.x.cpu().numpy(), host.x.ravel()), step
        assert np.array_equal(dev.v.cpu().numpy(), host.v.ravel()), step
        assert np.array_equal(dev.last["lam"].cpu().numpy().reshape(-1, 3), lo), step


@pytest.mark.gpu
def test_gpu_pile_contacts_equal_host_detection():
    """Device spatial hash + narrow phase + nodalization vs the host
    restatement (oracle/pile_host detect / nodalize) on the same (deformed, moving) state: every array bit-equal."""
    from paper_2201_09212_b200.pile import PileStepper
    from paper_2201_09212_b200.solver import SolverConfig

    dev = PileStepper(small_pile(nx_cubes=2, ny_cubes=2, layers=2, seed=9))
    for _ in range(3):
        dev.step(SolverConfig(residual_tol=1e-8, max_iters=100))
    pile = dev.pile
    pile.x = dev.x.cpu().numpy().reshape(-1, 3)
    pile.v = dev.v.cpu().numpy().reshape(-1, 3)
    hc, dc = H.contacts(pile), dev.device_contacts()
    assert (hc.n_ground, hc.n_face, hc.n_virtual) == (dc.n_ground, dc.n_face, dc.n_virtual)
    assert hc.n_face > 0 and hc.n_virtual > hc.n_face
    for name in ("col_i", "col_j", "frames", "phi", "mu"):
        assert np.array_equal(getattr(hc, name), getattr(dc, name)), name
    for name in ("indptr", "indices", "data"):
        assert np.array_equal(getattr(hc.jv, name), getattr(dc.jv, name)), name


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(4))
def test_gpu_pile_random_geometries(seed):
    """Random small piles (grid shape, resolution, gaps, jitter incl. z): the
    device step pipeline equals the host/oracle pipeline bit for bit over 4 steps."""
    from paper_2201_09212_b200.pile import PileStepper
    from paper_2201_09212_b200.solver import SolverConfig

    g = np.random.default_rng(40 + seed)
    kw = dict(nx_cubes=int(g.integers(1, 3)), ny_cubes=int(g.integers(1, 3)), layers=int(g.integers(2, 4)),
              nodes=int(g.integers(3, 6)), gap=float(g.choice([0.0, 1e-4])), jitter=float(g.choice([0.0, 5e-5, 2e-4])),
              gap_z=0.0, jitter_z=float(g.choice([0.0, 3e-5])), seed=int(g.integers(1000)), dt=5e-4,
              k_v=float(g.choice([1e2, 1e5])), mu=float(g.uniform(0.2, 0.8)))
    host = CubePile(**kw)
    dev = PileStepper(CubePile(**kw))
    prev = None
    faces = 0
    for step in range(4):
        pc, _, _, _, vo, lo, ro = _oracle_step(host, prev, 60)
        st = dev.step(SolverConfig(residual_tol=1e-8, max_iters=60))
        faces += pc.n_face
        assert (st["n_c"], st["n_face"], st["iterations"]) == (pc.n_c, pc.n_face, ro.iterations), (kw, step)
        H.advance(host, vo)
        prev = vo
        assert np.array_equal(dev.x.cpu().numpy(), host.x.ravel()), (kw, step)
        assert np.array_equal(dev.last["lam"].cpu().numpy().reshape(-1, 3), lo), (kw, step)
    assert faces > 0
