"""Virtual-node augmentation (reference
``augment_dynamics``, contacts.py:343-375).

CPU: the oracle restatement against golden vectors produced by the reference
itself (``tests/golden/make_golden_augment.py``). GPU (``-m gpu``): the device
augmentation (``vfpi_augment``) against the same goldens and against the
reference's scipy expression at configs[1] size — bit for bit, pattern and
values."""

import os

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import vfpi_oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = ["aug_rigid", "aug_face", "aug_none"]


def load(name):
    return dict(np.load(os.path.join(GOLD, name + ".npz")))


def jv_of(d):
    return sp.csr_matrix((d["jv_data"], d["jv_indices"], d["jv_indptr"]), shape=(int(d["jv_rows"]), int(d["n_o"])))


@pytest.mark.parametrize("name", CASES)
def test_oracle_augment_matches_reference(name):
    d = load(name)
    p, i, x, b = O.augment(int(d["n_o"]), d["a_indptr"], d["a_indices"], d["a_data"], d["b_o"], jv_of(d),
                           float(d["k_v"]))
    assert np.array_equal(p, d["out_indptr"])
    assert np.array_equal(i, d["out_indices"])
    assert np.array_equal(x, d["out_data"])
    assert np.array_equal(b, d["out_b"])


def test_golden_cases_exercise_the_stored_entry_rules():
    r = load("aug_rigid")
    # explicit zeros of A_o vanish in the top-left sum, J_v's zeros stay in the off-diagonal blocks
    assert (r["a_data"] == 0).any()
    n_o = int(r["n_o"])
    top = sp.csc_matrix((r["out_data"], r["out_indices"], r["out_indptr"]))[:n_o, :n_o]
    assert not (top.data == 0).any()
    assert (r["out_data"] == 0).any()
    # exact cancellations in J_v^T J_v: fewer top-left entries than the union of the patterns
    jv = jv_of(r)
    pat = jv.copy()
    pat.data = (pat.data != 0).astype(float)
    assert (jv.T @ jv).nnz < (pat.T @ pat).nnz
    f = load("aug_face")
    assert (f["jv_data"] == 0).any() and int(f["jv_rows"]) > 0


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_device_augment_matches_reference(name):
    from paper_2201_09212_b200.augment import augment_arrays

    d = load(name)
    p, i, x = augment_arrays(int(d["n_o"]), d["a_indptr"], d["a_indices"], d["a_data"], jv_of(d), float(d["k_v"]))
    assert np.array_equal(p, d["out_indptr"])
    assert np.array_equal(i, d["out_indices"])
    assert np.array_equal(x, d["out_data"])


@pytest.mark.gpu
def test_device_augment_dynamics_api():
    from paper_2201_09212_b200.augment import augment_dynamics
    from paper_2201_09212_b200.errors import DimensionMismatchError
    from paper_2201_09212_b200.system import Contact, NodalContactSet, SparseSymmetric

    d = load("aug_face")
    n_o = int(d["n_o"])
    a_o = SparseSymmetric(n_o, d["a_indptr"], d["a_indices"], d["a_data"])
    nv = int(d["jv_rows"]) // 3
    frame = np.eye(3)
    cs = [Contact("D", ("orig", 0), frame, 0.5, 0.0, slot_j=("virt", 1)), Contact("S", ("virt", 2), frame, 0.5, 0.0)]
    aug = augment_dynamics(a_o, d["b_o"], NodalContactSet(cs, nv, jv_of(d), float(d["k_v"])))
    assert aug.n == n_o + 3 * nv and aug.n_orig == n_o
    assert np.array_equal(aug.a.data, d["out_data"]) and np.array_equal(aug.b, d["out_b"])
    assert list(aug.col_i) == [0, n_o + 6] and list(aug.col_j) == [n_o + 3, -1]
    with pytest.raises(DimensionMismatchError):
        augment_dynamics(a_o, d["b_o"][:-1], NodalContactSet(cs, nv, jv_of(d), 1e5))


@pytest.mark.gpu
def test_device_augment_configs1_size():
    """Full configs[1] (4096 bodies, 32768 virtual nodes): device == scipy."""
    from paper_2201_09212_b200.scenes import rigid_contact_system

    host = rigid_contact_system()
    dev = rigid_contact_system(augment="device")
    assert np.array_equal(host.indptr, dev.indptr)
    assert np.array_equal(host.indices, dev.indices)
    assert np.array_equal(host.data, dev.data)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(12))
def test_device_augment_random_systems(seed):
    """Random A_o (explicit zeros included) and random J_v (random widths, exact
    zeros, exact cancellations, duplicate COO entries summed by the shim) --
    device augmentation == the reference expression, bit for bit."""
    from paper_2201_09212_b200.augment import augment_arrays

    g = np.random.default_rng(1000 + seed)
    n_o = int(g.integers(6, 90))
    a = sp.random(n_o, n_o, density=float(g.uniform(0.05, 0.4)), random_state=g, format="csc")
    a = (a + a.T + sp.identity(n_o)).tocsc()
    if seed % 3 == 0:  # explicit zeros in A_o
        a.data[g.random(a.nnz) < 0.2] = 0.0
    a.sort_indices()
    rows = int(g.integers(1, 30)) * 3
    nnz = int(g.integers(1, rows * 6))
    r = g.integers(0, rows, nnz)
    c = g.integers(0, n_o, nnz)
    v = np.where(g.random(nnz) < 0.2, 0.0, np.round(g.standard_normal(nnz) * 4) / 4)  # exact sums and zeros
    jv = sp.csr_matrix((v, (r, c)), shape=(rows, n_o))  # duplicates summed here, like nodalize's COO -> CSR
    kv = float(g.choice([1e5, 1e2, 3.0]))
    p, i, x = augment_arrays(n_o, a.indptr, a.indices, a.data, jv, kv)
    po, io, xo, _ = O.augment(n_o, a.indptr, a.indices, a.data, np.zeros(n_o), jv, kv)
    assert np.array_equal(p, po) and np.array_equal(i, io) and np.array_equal(x, xo)


@pytest.mark.gpu
def test_device_augment_rejects_non_canonical_jv():
    """vfpi_augment_device validates J_v (columns in range, increasing per row)."""
    import ctypes as C

    import torch

    from paper_2201_09212_b200 import _lib

    n_o = 6
    a = sp.identity(n_o, format="csc")
    up = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x, dtype=dt)).cuda()  # noqa: E731
    ap, ai, ax = up(a.indptr, np.int32), up(a.indices, np.int32), up(a.data, np.float64)
    for cols in ([0, 7, 1], [2, 1, 3]):  # out of range / not increasing
        jp, ji, jx = up([0, 3, 3, 3], np.int32), up(cols, np.int32), up([1.0, 1.0, 1.0], np.float64)
        h = _lib.handle(0)
        inp = _lib.VfpiAugmentInput(n_o, 3, a.nnz, C.cast(ap.data_ptr(), _lib._i32p), C.cast(ai.data_ptr(), _lib._i32p),
                                    C.cast(ax.data_ptr(), _lib._f64p), 3, C.cast(jp.data_ptr(), _lib._i32p),
                                    C.cast(ji.data_ptr(), _lib._i32p), C.cast(jx.data_ptr(), _lib._f64p), 1e5)
        out = _lib.VfpiAugmented()
        assert h.L.vfpi_augment_device(h.h, C.byref(inp), C.byref(out), None) == _lib.BAD_ARGUMENT
