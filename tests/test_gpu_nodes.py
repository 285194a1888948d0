"""The node-block SELL scene kernel (csrc/vfpi_nodes.cu) against the row-SELL
scene kernel and the CPU oracle: FEM batches stepped through contact with
either kernel end in bit-identical states with the same iteration counts,
for every operator, Chebyshev, and the fixed-alpha step."""

import numpy as np
import pytest

from oracle import fem_host as F

pytestmark = pytest.mark.gpu


def _cubes(nx, n, seed):
    from paper_2201_09212_b200.scenes import FemCube

    g = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        c = FemCube(nx=nx, E=float(g.uniform(5e4, 2e5)), drop=float(g.uniform(0.0005, 0.004)),
                    yaw=float(g.uniform(0, 2 * np.pi)))
        out.append(c)
    return out


def test_node_template_covers_every_block():
    from paper_2201_09212_b200.fembatch import node_block_template
    from paper_2201_09212_b200.scenes import FemCube

    c = FemCube(nx=7, yaw=0.3)
    order, soff, bcols = node_block_template(c.K.indptr, c.K.indices, c.n)
    assert sorted(order.tolist()) == list(range(c.n // 3))
    nb = int((bcols >= 0).sum())
    K = c.K.tocoo()
    assert nb == np.unique((K.row // 3) * (c.n // 3) + K.col // 3).size
    w = np.diff(soff)
    assert (w[:-1] >= w[1:]).all()  # decreasing block counts -> decreasing slice widths


@pytest.mark.parametrize("kw", [dict(), dict(chebyshev=True), dict(operator="proximal"),
                                dict(operator="strict-anisotropic"), dict(step_strategy="fixed-alpha")])
def test_node_kernel_equals_row_kernel(kw):
    from paper_2201_09212_b200.fembatch import FemBatch
    from paper_2201_09212_b200.solver import SolverConfig

    cfg = SolverConfig(residual_tol=1e-8, max_iters=400, **kw)
    a = FemBatch(_cubes(6, 12, 3), node_layout=True)
    b = FemBatch(_cubes(6, 12, 3), node_layout=False)
    assert a.node_kernel and not b.node_kernel
    contacts = 0
    for step in range(40):
        sa, sb = a.step(cfg, per_scene=True), b.step(cfg, per_scene=True)
        assert sa["node_kernel"] and not sb["node_kernel"]
        assert sa["contacts"] == sb["contacts"], step
        contacts += sa["contacts"]
        assert np.array_equal(sa["iterations_per_scene"], sb["iterations_per_scene"]), step
        assert sa["diverged_scenes"] == sb["diverged_scenes"]
    assert contacts > 0
    xa, va = a.state()
    xb, vb = b.state()
    if kw.get("chebyshev"):
        # Chebyshev's rho = theta_l / theta_{l-1} depends on the reduction order
        # of theta (the kernels visit rows in different orders; the reference's
        # is an OpenBLAS dot): last-bit differences in nu, so tolerance-equal
        assert np.linalg.norm(xa - xb) <= 1e-12 * np.linalg.norm(xb)
        assert np.linalg.norm(va - vb) <= 1e-9 * np.linalg.norm(vb)
    else:
        assert np.array_equal(xa, xb) and np.array_equal(va, vb)
    a.close()
    b.close()


def test_node_kernel_matches_oracle_pipeline():
    from paper_2201_09212_b200.fembatch import FemBatch
    from paper_2201_09212_b200.solver import SolverConfig

    steps = 30
    fb = FemBatch(_cubes(5, 6, 11))
    assert fb.node_kernel
    cfg = SolverConfig(residual_tol=1e-8, max_iters=500)
    its = [fb.step(cfg, per_scene=True)["iterations_per_scene"].tolist() for _ in range(steps)]
    x, v = fb.state()
    for k, c in enumerate(_cubes(5, 6, 11)):
        rec = []
        F.oracle_steps(c, steps, residual_tol=1e-8, max_iters=500, record=rec)
        assert [r["iterations"] for r in rec] == [row[k] for row in its], k
        assert sum(r["n_c"] for r in rec) > 0
        assert np.array_equal(x[k], c.x) and np.array_equal(v[k], c.v), k


def _grid_case(case):
    from oracle import pile_host as H
    from paper_2201_09212_b200.pile import CubePile
    from paper_2201_09212_b200.scenes import HeightfieldBlock, rigid_contact_system

    if case == "rigid":
        return rigid_contact_system(96, 300, seed=4, k_v=1e3)
    if case == "heightfield":
        return F.heightfield_system(HeightfieldBlock(nx=10))
    pile = CubePile(nx_cubes=2, ny_cubes=1, layers=2, nodes=4, gap=0.0, jitter=0.00005, seed=5, dt=5e-4)
    return H.system(pile)


@pytest.mark.parametrize("case", ["rigid", "heightfield", "pile"])
@pytest.mark.parametrize("cheb", [False, True])
def test_grid_node_kernel_equals_row_streaming_kernel(case, cheb):
    """Single systems on the global-memory path: the node-block grid kernel
    against the row-SELL streaming kernel (and the oracle, plain V-FPI)."""
    from oracle import vfpi_oracle as O
    from paper_2201_09212_b200 import _lib
    from paper_2201_09212_b200.solver import SolverConfig, solve_packed

    ps = _grid_case(case)
    cfg = SolverConfig(residual_tol=1e-9, max_iters=150, chebyshev=cheb)
    warm = np.zeros(ps.n)
    h = _lib.handle()
    h.set_kernel("streaming")
    try:
        h.set_node_kernel(True)
        v1, l1, r1 = solve_packed(ps, cfg, warm)
        assert h.last_layout()["node_kernel"]
        h.set_node_kernel(False)
        v2, l2, r2 = solve_packed(ps, cfg, warm)
        assert not h.last_layout()["node_kernel"]
    finally:
        h.set_kernel("auto")
        h.set_node_kernel(True)
    assert r1.iterations == r2.iterations and r1.converged == r2.converged
    if cheb:
        # rho = theta_l / theta_{l-1}: last-bit differences of theta (reduction
        # order) reach v and lam through nu; stiff virtual-node systems amplify
        # them (the reference moves 1e-1 under a 1e-15 input change)
        tol = 1e-9 if case == "heightfield" else 1e-6
        assert np.linalg.norm(v1 - v2) <= tol * np.linalg.norm(v2)
        assert np.linalg.norm(l1 - l2) <= tol * max(np.linalg.norm(l2), 1e-300)
    else:
        assert np.array_equal(v1, v2) and np.array_equal(l1, l2)
        s = O.System(ps.n, ps.indptr, ps.indices, ps.data, ps.b, ps.col_i.astype(np.int64),
                     ps.col_j.astype(np.int64), ps.frames.reshape(-1, 3, 3), ps.mu, ps.mu2, ps.phi)
        vo, lo, ro = O.solve(s, O.Config(residual_tol=1e-9, max_iters=150), warm)
        assert ro.iterations == r1.iterations
        assert np.array_equal(v1, vo) and np.array_equal(l1, lo)


@pytest.mark.parametrize("kw", [dict(), dict(operator="proximal"), dict(chebyshev=True)])
def test_cluster_per_scene_equals_one_cta_per_scene(kw):
    """A small batch (16 scenes) runs one thread-block cluster per scene (the
    scene's node slices split over the cluster's CTAs, partials summed over
    distributed shared memory); it must equal the one-CTA-per-scene kernel."""
    from paper_2201_09212_b200 import _lib
    from paper_2201_09212_b200.fembatch import FemBatch
    from paper_2201_09212_b200.solver import SolverConfig

    h = _lib.handle()
    cfg = SolverConfig(residual_tol=1e-8, max_iters=300, **kw)
    try:
        h.set_node_cluster(True)
        a = FemBatch(_cubes(6, 16, 5))
        h.set_node_cluster(False)
        b = FemBatch(_cubes(6, 16, 5))
    finally:
        h.set_node_cluster(True)
    # the small batch really runs on clusters, and both layouts take their block
    # columns from the batch's template: no descriptor stream, the same bytes
    # per scene iteration (vfpi_fem_layout_info)
    assert a.cluster > 1 and b.cluster == 1
    assert a.layout_bytes_per_scene_iter == b.layout_bytes_per_scene_iter > 0
    contacts = 0
    for step in range(30):
        sa, sb = a.step(cfg, per_scene=True), b.step(cfg, per_scene=True)
        assert sa["node_kernel"] and sb["node_kernel"]
        assert sa["contacts"] == sb["contacts"], step
        contacts += sa["contacts"]
        assert np.array_equal(sa["iterations_per_scene"], sb["iterations_per_scene"]), step
    assert contacts > 0
    xa, va = a.state()
    xb, vb = b.state()
    if kw.get("chebyshev"):
        assert np.linalg.norm(va - vb) <= 1e-9 * np.linalg.norm(vb)
    else:
        assert np.array_equal(xa, xb) and np.array_equal(va, vb)
    a.close()
    b.close()


@pytest.mark.parametrize("kw", [dict(), dict(chebyshev=True), dict(step_strategy="fixed-alpha", fixed_alpha=1e3)])
@pytest.mark.parametrize("cluster", [True, False])
def test_device_run_equals_step_loop(kw, cluster):
    """FemBatch.run (vfpi_fem_run: no host round trip per step, the diverged-scene
    fallback decided on the device) equals the same number of FemBatch.step calls."""
    from paper_2201_09212_b200 import _lib
    from paper_2201_09212_b200.fembatch import FemBatch
    from paper_2201_09212_b200.solver import SolverConfig

    h = _lib.handle()
    cfg = SolverConfig(residual_tol=1e-8, max_iters=200, **kw)
    steps = 25
    try:
        h.set_node_cluster(cluster)
        a = FemBatch(_cubes(6, 10, 8))
        b = FemBatch(_cubes(6, 10, 8))
    finally:
        h.set_node_cluster(True)
    r = a.run(cfg, steps, per_step=True)
    assert r["host_synced"] == 0
    its, cts, div = [], [], 0
    for _ in range(steps):
        st = b.step(cfg, per_scene=True)
        its.append(st["iterations_per_scene"])
        cts.append(st["contacts"])
        div += st["diverged_scenes"]
    assert np.array_equal(r["iterations_per_step"], np.array(its))
    assert np.array_equal(r["contacts_per_step"], np.array(cts)) and sum(cts) > 0
    assert r["diverged_scene_steps"] == div
    if kw.get("step_strategy") == "fixed-alpha":
        assert div > 0
    xa, va = a.state()
    xb, vb = b.state()
    assert np.array_equal(xa, xb) and np.array_equal(va, vb)
    a.close()
    b.close()
