"""Nodalization (reference ``nodalize``, contacts.py:271-321): the oracle
restatement against the reference's own output on mixed rigid / node / static
sides (CPU), and the device nodalization ``vfpi_nodalize_device`` against the
same golden (-m gpu) -- slots, virtual nodes, J_v (pattern, values, explicit
zeros), frames and phi bit for bit."""

import os

import numpy as np
import pytest

from oracle import vfpi_oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "nodalize_mixed.npz")


def load():
    return dict(np.load(GOLD))


def _check(d, col_i, col_j, frames, phi, mu, mu2, jv, nv):
    assert nv == int(d["out_n_virtual"])
    assert np.array_equal(col_i, d["out_col_i"]) and np.array_equal(col_j, d["out_col_j"])
    assert np.array_equal(np.asarray(frames).reshape(-1), d["out_frames"])
    assert np.array_equal(phi, d["out_phi"])
    assert np.array_equal(mu, d["out_mu"]) and np.array_equal(mu2, d["out_mu2"])
    assert np.array_equal(jv.indptr, d["out_jv_indptr"]) and np.array_equal(jv.indices, d["out_jv_indices"])
    assert np.array_equal(jv.data, d["out_jv_data"])
    assert np.array_equal(np.signbit(jv.data), np.signbit(d["out_jv_data"]))


def test_oracle_nodalize_matches_reference():
    d = load()
    out = O.nodalize(d["first_kind"], d["first_ref"], d["second_kind"], d["second_ref"], d["point"], d["normal"],
                     d["depth"], d["q"], d["v"], d["body_q"], d["body_v"], d["v"].shape[0], float(d["mu"]),
                     float(d["mu2"]), float(d["beta"]), float(d["dt"]), float(d["e_rest"]), float(d["thr"]))
    _check(d, *out)


def test_golden_exercises_every_side_kind():
    d = load()
    assert set(d["first_kind"].tolist()) == {0, 1} and set(d["second_kind"].tolist()) == {-1, 0, 1}
    # more virtual nodes than rigid sides: some nodes carry a second contact
    rigid_sides = int((d["first_kind"] == 1).sum() + (d["second_kind"] == 1).sum())
    assert int(d["out_n_virtual"]) > rigid_sides
    # restitution branch taken somewhere
    assert not np.array_equal(d["out_phi"], -(float(d["beta"]) / float(d["dt"])) * d["depth"])


@pytest.mark.gpu
def test_device_nodalize_matches_reference():
    from paper_2201_09212_b200.nodalize import nodalize_arrays

    d = load()
    out = nodalize_arrays(d["first_kind"], d["first_ref"], d["second_kind"], d["second_ref"], d["point"],
                          d["normal"], d["depth"], d["q"], d["v"], d["body_q"], d["body_v"], float(d["mu"]),
                          float(d["mu2"]), float(d["beta"]), float(d["dt"]), float(d["e_rest"]), float(d["thr"]))
    _check(d, out["col_i"], out["col_j"], out["frames"], out["phi"], out["mu"], out["mu2"], out["jv"],
           out["n_virtual"])


def _raw_from_golden(d):
    from collections import namedtuple

    Raw = namedtuple("Raw", "point normal depth first second")
    names = {0: "node", 1: "rigid", -1: "static"}
    out = []
    for m in range(d["first_kind"].shape[0]):
        def side(kind, ref):
            if kind == -1:
                return ("static",)
            return ("node", int(ref)) if kind == 0 else ("rigid", int(ref), m)
        out.append(Raw(d["point"][m], d["normal"][m], float(d["depth"][m]), side(int(d["first_kind"][m]),
                   d["first_ref"][m]), side(int(d["second_kind"][m]), d["second_ref"][m])))
        assert names[int(d["first_kind"][m])] == out[-1].first[0]
    return out


@pytest.mark.gpu
def test_device_chain_nodalize_augment_solve():
    """Reference per-step restructuring on the device: nodalize (drop-in API,
    reference objects in) -> augment_dynamics -> solve_vfpi, against the oracle
    chain on the same inputs; bit-equal v and lam."""
    from collections import namedtuple

    import scipy.sparse as sp

    from paper_2201_09212_b200.augment import augment_dynamics
    from paper_2201_09212_b200.nodalize import nodalize
    from paper_2201_09212_b200.solver import SolverConfig, solve_vfpi
    from paper_2201_09212_b200.system import SparseSymmetric

    d = load()
    State = namedtuple("State", "q v dt")
    BodyT = namedtuple("BodyT", "q_offset v_offset")
    Stab = namedtuple("Stab", "beta_err e_rest v_rest_threshold dt")
    bodies = [BodyT(int(a), int(b)) for a, b in zip(d["body_q"], d["body_v"])]
    state = State(d["q"], d["v"], float(d["dt"]))
    stab = Stab(float(d["beta"]), float(d["e_rest"]), float(d["thr"]), float(d["dt"]))
    nodal = nodalize(_raw_from_golden(d), state, bodies, float(d["k_v"]), float(d["mu"]), float(d["mu2"]), stab)
    assert nodal.n_virtual == int(d["out_n_virtual"])
    assert np.array_equal(np.array([c.phi_n for c in nodal.contacts]), d["out_phi"])
    n_o = d["v"].shape[0]
    rng = np.random.default_rng(3)
    blocks = []
    for k in range(0, n_o, 3):
        m = rng.standard_normal((3, 3))
        blocks.append(m @ m.T + 3.0 * np.eye(3))
    a_o = SparseSymmetric.from_scipy(sp.block_diag([sp.csc_matrix(bk) for bk in blocks], format="csc"))
    b_o = rng.standard_normal(n_o)
    aug = augment_dynamics(a_o, b_o, nodal)
    cfg = SolverConfig(residual_tol=1e-10, max_iters=80)
    v, lam, rep = solve_vfpi(aug, cfg, np.zeros(aug.n))
    # oracle chain
    oc = O.nodalize(d["first_kind"], d["first_ref"], d["second_kind"], d["second_ref"], d["point"], d["normal"],
                    d["depth"], d["q"], d["v"], d["body_q"], d["body_v"], n_o, float(d["mu"]), float(d["mu2"]),
                    float(d["beta"]), float(d["dt"]), float(d["e_rest"]), float(d["thr"]))
    col_i, col_j, frames, phi, mu, mu2, jv, nv = oc
    p, i, x, b = O.augment(n_o, a_o.indptr, a_o.indices, a_o.data, b_o, jv, float(d["k_v"]))
    s = O.System(n_o + 3 * nv, p, i, x, b, col_i, col_j, frames, mu, mu2, phi)
    vo, lo, ro = O.solve(s, O.Config(residual_tol=1e-10, max_iters=80), np.zeros(n_o + 3 * nv))
    assert np.array_equal(aug.a.data, x) and np.array_equal(aug.a.indices, i)
    assert rep.iterations == ro.iterations
    assert np.array_equal(v, vo) and np.array_equal(lam, lo)


@pytest.mark.gpu
def test_device_nodalize_edge_cases():
    """No contacts; a zero normal raises like contact_frame (contacts.py:139-140)."""
    from paper_2201_09212_b200.errors import DeviceError
    from paper_2201_09212_b200.nodalize import nodalize_arrays

    d = load()
    e = np.zeros(0, np.int32)
    out = nodalize_arrays(e, e, e, e, np.zeros((0, 3)), np.zeros((0, 3)), np.zeros(0), d["q"], d["v"], d["body_q"],
                          d["body_v"])
    assert out["n_virtual"] == 0 and out["col_i"].size == 0 and out["jv"].shape == (0, d["v"].shape[0])
    with pytest.raises((ValueError, DeviceError)):
        nodalize_arrays(np.array([0], np.int32), np.array([0], np.int32), np.array([-1], np.int32),
                        np.array([-1], np.int32), np.zeros((1, 3)), np.zeros((1, 3)), np.zeros(1), d["q"], d["v"],
                        d["body_q"], d["body_v"])


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(8))
def test_device_nodalize_random_contacts(seed):
    """Random raw contact sets (every side kind, repeated nodes, moving bodies,
    restitution on) -- device nodalization == the oracle restatement bit for bit."""
    from paper_2201_09212_b200.nodalize import nodalize_arrays

    g = np.random.default_rng(500 + seed)
    n_rigid, n_part = int(g.integers(1, 8)), int(g.integers(2, 12))
    body_q, body_v, q, v = [], [], [], []
    qo = vo = 0
    for _ in range(n_rigid):
        body_q.append(qo)
        body_v.append(vo)
        quat = g.standard_normal(4)
        q += list(g.uniform(-1, 1, 3)) + list(quat / np.linalg.norm(quat))
        v += list(g.standard_normal(6))
        qo += 7
        vo += 6
    for _ in range(n_part):
        body_q.append(qo)
        body_v.append(vo)
        q += list(g.uniform(-1, 1, 3))
        v += list(g.standard_normal(3) * 0.1)
        qo += 3
        vo += 3
    q, v = np.array(q), np.array(v)
    n_c = int(g.integers(1, 50))
    fk = g.integers(0, 2, n_c).astype(np.int32)
    sk = g.integers(-1, 2, n_c).astype(np.int32)
    fr = np.where(fk == 0, [body_v[n_rigid + int(g.integers(n_part))] for _ in range(n_c)],
                  g.integers(0, n_rigid, n_c)).astype(np.int32)
    sr = np.where(sk == 0, [body_v[n_rigid + int(g.integers(n_part))] for _ in range(n_c)],
                  np.where(sk == 1, g.integers(0, n_rigid, n_c), -1)).astype(np.int32)
    pt = g.uniform(-1, 1, (n_c, 3))
    nrm = g.standard_normal((n_c, 3)) * g.choice([1.0, 3.0], (n_c, 1))
    depth = np.abs(g.normal(0, 1e-3, n_c))
    args = (fk, fr, sk, sr, pt, nrm, depth, q, v, np.array(body_q, np.int32), np.array(body_v, np.int32))
    prm = (0.4, None if seed % 2 else 0.25, 0.2, 1e-3, 0.5, 0.01)
    out = nodalize_arrays(*args, *prm)
    ci, cj, frames, phi, mu, mu2, jv, nv = O.nodalize(*args, v.shape[0], *prm)
    assert out["n_virtual"] == nv
    assert np.array_equal(out["col_i"], ci) and np.array_equal(out["col_j"], cj)
    assert np.array_equal(out["frames"], frames) and np.array_equal(out["phi"], phi)
    assert np.array_equal(out["mu"], mu) and np.array_equal(out["mu2"], mu2)
    assert np.array_equal(out["jv"].indptr, jv.indptr) and np.array_equal(out["jv"].indices, jv.indices)
    assert np.array_equal(out["jv"].data, jv.data) and np.array_equal(np.signbit(out["jv"].data), np.signbit(jv.data))


@pytest.mark.gpu
def test_device_nodalize_rejects_bad_sides():
    """Out-of-range node offsets / body ids and a static first side are refused
    before any output is written."""
    from paper_2201_09212_b200.nodalize import nodalize_arrays

    d = load()
    base = dict(point=np.zeros((1, 3)), normal=np.array([[0.0, 0.0, 1.0]]), depth=np.zeros(1))
    for fk, fr, sk, sr in ((0, d["v"].shape[0], -1, -1), (1, len(d["body_q"]), -1, -1), (-1, 0, -1, -1),
                           (0, 0, 1, -5)):
        with pytest.raises(ValueError):
            nodalize_arrays(np.array([fk], np.int32), np.array([fr], np.int32), np.array([sk], np.int32),
                            np.array([sr], np.int32), base["point"], base["normal"], base["depth"], d["q"], d["v"],
                            d["body_q"], d["body_v"])
