"""Pin the CPU oracle against golden vectors produced by the reference itself.

CPU only. The oracle is trusted as the GPU checker only because these pass.
"""

import numpy as np
import pytest

from golden_cases import load, names, oracle_config, oracle_system
from oracle import vfpi_oracle as O

CASES = names()


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(1.0, np.linalg.norm(b)))


@pytest.mark.parametrize("name", CASES)
def test_sparse_ops_bit_exact(name):
    d = load(name)
    s = oracle_system(d)
    x = d["op_x"]
    assert np.array_equal(O.spmv(s, x), d["op_spmv"])
    # the CUDA kernel's order (sequential per CSR row, FMA-free) equals scipy's
    assert np.array_equal(O.spmv_rowseq(s, x), d["op_spmv"])
    assert np.array_equal(O.row_norms_sq(s), d["op_rns"])
    assert np.array_equal(O.diagonal(s), d["op_diag"])
    if "op_w_strict" in d:
        assert np.array_equal(O.step_matrix_frobenius(s, False), d["op_w_strict"])
        assert np.array_equal(O.step_matrix_frobenius(s, True), d["op_w_prox"])


@pytest.mark.parametrize("name", [c for c in CASES if load(c)["col_i"].size])
def test_contact_ops_bit_exact(name):
    d = load(name)
    s = oracle_system(d)
    n_c = s.n_c
    cfg = d["cfg"]
    w = O.step_matrix_frobenius(s, cfg["operator"] == "proximal")
    gam = O.surrogate_gamma(s, w, cfg["omega"])
    assert np.array_equal(gam, d["op_gamma"])
    assert np.array_equal(O.apply_jc(s, d["op_x"]).reshape(-1), d["op_jc"])
    assert np.array_equal(O.apply_jc_t(s, d["op_lam"].reshape(n_c, 3)), d["op_jct"])
    eta = d["op_eta"].reshape(n_c, 3)
    for op in ("strict", "proximal"):
        got = O.oneshot(gam, eta, s.phi, s.mu, s.mu2, op).reshape(-1)
        assert np.array_equal(got, d["op_oneshot_" + op], equal_nan=True), op
    got = O.oneshot(gam, eta, s.phi, s.mu, s.mu2, "strict-anisotropic").reshape(-1)
    assert np.array_equal(got, d["op_oneshot_strict_anisotropic"], equal_nan=True)
    assert np.array_equal(O.inverse_contact(s, d["op_x"], 1e-3).reshape(-1), d["op_inverse"])


@pytest.mark.parametrize("name", CASES)
def test_solve_matches_reference(name):
    d = load(name)
    s = oracle_system(d)
    cfg = oracle_config(d)
    w_cached = d.get("w_cached")
    if d["out_diverged"]:
        with np.errstate(over="ignore", invalid="ignore"):
            with pytest.raises(O.OracleDivergence) as exc:
                O.solve(s, cfg, d["warm"], w_cached)
        tr = np.array(exc.value.residual_trace)
        assert len(tr) == int(d["out_iterations"])
        fin = np.isfinite(d["out_trace"])
        assert np.allclose(tr[fin], d["out_trace"][fin], rtol=1e-9)
        return
    with np.errstate(over="ignore", invalid="ignore"):
        v, lam, rep = O.solve(s, cfg, d["warm"], w_cached)
    assert rep.iterations == int(d["out_iterations"])
    assert rep.converged == bool(d["out_converged"])
    assert rel(v, d["out_v"]) <= 1e-12
    assert rel(lam.reshape(-1), d["out_lam"]) <= 1e-12
    assert np.allclose(rep.residual_trace, d["out_trace"], rtol=1e-9, atol=1e-300, equal_nan=True)
    assert np.isclose(rep.consistency, float(d["out_consistency"]), rtol=1e-6, atol=1e-14, equal_nan=True)
    if s.n_c:
        assert np.allclose(rep.scc_residuals, d["out_scc"], rtol=1e-9, atol=1e-14, equal_nan=True)


def test_pairwise_sum_matches_numpy():
    g = np.random.default_rng(0)
    for n in (0, 1, 5, 7, 8, 9, 16, 17, 127, 128, 129, 300, 1000):
        x = g.standard_normal(n) * 10.0 ** g.integers(-6, 6, n)
        assert O.pairwise_sum(x) == (np.sum(x) if n else 0.0)
        if n:
            assert np.add.reduceat(x, [0])[0] == x[0] + O.pairwise_sum(x[1:])
