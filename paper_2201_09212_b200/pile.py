"""configs[4]: a pile of deformable cubes with node-to-face contacts
(SURVEY §8(f) items 2-3).

The reference has no FEM and no face-side contacts: ``detect_contacts``
(``contacts.py:159-227``) pairs sphere proxies through a KD-tree and
``_slot_and_jv`` (``:242-268``) resolves only ``node`` and ``rigid`` sides.
This module keeps the reference's pipeline and adds the missing pieces the
way the reference would write them:

* **geometry** -- ``n_x x n_y x layers`` copies of the ``scenes.FemCube``
  linear-tet cube (configs[0] material), placed on a grid with seeded jitter;
  A_o, K, M are block diagonal (one block per cube, the cube's own arrays);
* **broad phase** -- a spatial hash: every surface triangle is entered in the
  cells (edge ``2h``) its bounding box, grown by the search distance, overlaps;
  every surface node looks up its own cell (sort + binary search, no Python
  loop over contacts);
* **narrow phase** -- one pass (the classic slave-node / master-face split,
  so two coincident surfaces are never constrained from both sides): node
  ``p`` of cube A against triangle ``(a, b, c)`` of cube B < A (cubes are
  numbered layer by layer, so upper nodes meet lower faces): signed distance ``d = (p - a).n`` along B's outward normal,
  ``-h/2 < d < margin`` and the projection inside the triangle (barycentric
  weights ``w >= 0``); one contact per node, the candidate with the largest
  ``d``; ground contacts (plane ``z = 0``) as in ``scenes.FemCube``;
* **nodalize** -- ``contacts.py:271-321`` with a third side kind, ``face``:
  a virtual node tied to the triangle's three nodes by ``J_v = [w0 I, w1 I,
  w2 I]`` (three 3x3 blocks, stored entry by entry as ``nodalize`` stores its
  blocks); a node's second contact moves to an identity virtual node
  (``contacts.py:249-255``); plane contacts come first, as in
  ``detect_contacts``; frames ``contact_frame(n)``, ``phi`` from
  ``stabilization_term`` (``:230-239``);
* **augmentation** -- ``augment.augment_arrays`` (device, bit-identical to the
  reference's ``augment_dynamics``).

``PileStepper`` runs every piece on the device; ``oracle/pile_host.py``
holds their host restatement (the checker the tests compare against).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .scenes import FemCube, _tets
from .system import PackedSystem, make_packed


def surface_triangles(nx: int, X: np.ndarray) -> np.ndarray:
    """Boundary faces of the 5-tet hex split, oriented outward (T, 3)."""
    tets = _tets(nx)
    faces = np.concatenate([tets[:, [1, 2, 3]], tets[:, [0, 2, 3]], tets[:, [0, 1, 3]], tets[:, [0, 1, 2]]])
    opp = np.concatenate([tets[:, 0], tets[:, 1], tets[:, 2], tets[:, 3]])
    key = np.sort(faces, axis=1)
    _, inv, cnt = np.unique(key, axis=0, return_inverse=True, return_counts=True)
    bnd = cnt[inv.ravel()] == 1
    f, o = faces[bnd].copy(), opp[bnd]
    nrm = np.cross(X[f[:, 1]] - X[f[:, 0]], X[f[:, 2]] - X[f[:, 0]])
    inward = np.einsum("ij,ij->i", nrm, X[o] - X[f[:, 0]]) > 0
    f[inward, 1], f[inward, 2] = f[inward, 2], f[inward, 1].copy()
    return f


@dataclass
class PileContacts:
    """Nodalized contacts of one step (``NodalContactSet`` in flat arrays)."""

    col_i: np.ndarray
    col_j: np.ndarray
    frames: np.ndarray  # (n_c, 3, 3)
    phi: np.ndarray
    mu: np.ndarray
    jv: sp.csr_matrix   # (3 n_virtual, n_o)
    n_ground: int
    n_face: int

    @property
    def n_c(self) -> int:
        return int(self.col_i.shape[0])

    @property
    def n_virtual(self) -> int:
        return int(self.jv.shape[0]) // 3


class CubePile:
    """``nx_cubes x ny_cubes x layers`` FEM cubes of ``nodes^3`` nodes (configs[4]:
    8 x 8 x 4, 16^3, mu 0.6, dt 5e-4; small sizes for parity tests)."""

    def __init__(self, nx_cubes=8, ny_cubes=8, layers=4, nodes=16, side=0.1, gap=0.005, jitter=0.002, seed=0,
                 E=1e5, nu=0.3, rho=1000.0, dt=5e-4, mu=0.6, gravity=-9.81, margin=1e-4, beta_err=0.2,
                 e_rest=0.0, rest_threshold=0.01, k_v=1e5, gap_z=None, jitter_z=None):
        """``gap`` / ``jitter``: lateral spacing and U[-jitter, jitter] offsets in
        x and y; ``gap_z`` / ``jitter_z`` (default: the lateral values) the same
        between layers and above the plane."""
        self.dt, self.mu, self.margin, self.k_v = dt, mu, margin, k_v
        self.beta, self.e_rest, self.thr = beta_err, e_rest, rest_threshold
        self.h = side / (nodes - 1)
        cube = FemCube(nx=nodes, side=side, E=E, nu=nu, rho=rho, drop=0.0, dt=dt, mu=mu, gravity=gravity,
                       margin=margin, beta_err=beta_err, e_rest=e_rest, rest_threshold=rest_threshold)
        self.cube = cube
        nc = nx_cubes * ny_cubes * layers
        self.n_cubes, self.nn_cube = nc, nodes ** 3
        rng = np.random.default_rng(seed)
        gz = gap if gap_z is None else gap_z
        jz = jitter if jitter_z is None else jitter_z
        pitch = side + gap
        ix, iy, iz = np.meshgrid(np.arange(nx_cubes), np.arange(ny_cubes), np.arange(layers), indexing="ij")
        base = np.stack([ix.ravel() * pitch, iy.ravel() * pitch, gz + iz.ravel() * (side + gz)], axis=1)
        order = np.lexsort((base[:, 0], base[:, 1], base[:, 2]))  # layer-major cube order
        jit = rng.uniform(-1.0, 1.0, (nc, 3)) * np.array([jitter, jitter, jz])
        base = base[order] + jit
        Xt = cube.X - np.array([0.0, 0.0, 0.0])
        self.X = (Xt[None, :, :] + base[:, None, :]).reshape(-1, 3)
        self.x = self.X.copy()
        self.v = np.zeros_like(self.X)
        self.n = 3 * self.X.shape[0]
        self.node_cube = np.repeat(np.arange(nc), self.nn_cube)
        tri_t = surface_triangles(nodes, cube.X)
        self.tris = (tri_t[None, :, :] + (self.nn_cube * np.arange(nc))[:, None, None]).reshape(-1, 3)
        self.tri_cube = np.repeat(np.arange(nc), tri_t.shape[0])
        surf_t = np.unique(tri_t)
        self.surf = (surf_t[None, :] + (self.nn_cube * np.arange(nc))[:, None]).ravel()
        self.m = np.tile(cube.m, nc)
        self.gravity = np.tile(cube.gravity, nc)
        A, K = cube.A, cube.K.tocsr()
        K.sort_indices()
        self.a_indptr, self.a_indices, self.a_data = _tile_compressed(A, nc)
        self.k_indptr, self.k_indices, self.k_data = _tile_compressed(K, nc)

    def node_body_i32(self):
        return self.node_cube.astype(np.int32)



def _lib_cuda_copy(t, src_ptr, n, dt):
    """Copy n elements of a device pointer into tensor t (device to device)."""
    import ctypes as C

    from . import _lib

    nbytes = n * t.element_size()
    _lib.lib().vfpi_memcpy_d2d(C.c_void_p(t.data_ptr()), C.cast(src_ptr, C.c_void_p), C.c_int64(nbytes))


def _tile_compressed(m, copies: int):
    """Compressed arrays of ``copies`` diagonal copies of ``m`` (int32 indices)."""
    nnz, dim = m.nnz, m.shape[0]
    if copies * nnz >= 2 ** 31:
        raise ValueError("pile: more than 2^31 stored entries")
    ptr = (m.indptr[1:][None, :].astype(np.int64) + nnz * np.arange(copies, dtype=np.int64)[:, None]).ravel()
    ptr = np.concatenate([[0], ptr]).astype(np.int32)
    idx = (m.indices[None, :].astype(np.int32) + (dim * np.arange(copies, dtype=np.int32))[:, None]).ravel()
    return ptr, idx, np.tile(m.data, copies)


class PileStepper:
    """A ``CubePile`` stepped with its state in device memory (configs[4]).

    Per step, on the device: contact detection + nodalization
    (``vfpi_pile_contacts_device``; its host restatement, the checker, is
    ``oracle/pile_host.py``), b (``vfpi_fem_rhs_sell_device``,
    K packed once as SELL-32),
    the augmented matrix (``vfpi_augment_device``), the warm start
    (``vfpi_csr_matvec_device``, ``harness._warm_velocity``), the V-FPI solve
    (``vfpi_solve_device``) and the midpoint integration (``vfpi_advance_device``).
    A_o and K stay resident; torch tensors are plain device memory here."""

    def __init__(self, pile: CubePile, device: int | None = None):
        import torch

        from . import _lib

        self.h = _lib.handle(device)
        self.pile, self.device = pile, self.h.device
        self.dev = torch.device("cuda", self.device)
        up = lambda a, dt=None: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(self.dev)  # noqa: E731
        self.a = (up(pile.a_indptr, np.int32), up(pile.a_indices, np.int32), up(pile.a_data, np.float64))
        self.k = (up(pile.k_indptr, np.int64), up(pile.k_indices, np.int32), up(pile.k_data, np.float64))
        # K packed once as SELL-32 for the per-step right-hand side (coalesced stream)
        import ctypes as C

        from .solver import _raise_for

        nsl = (pile.n + 31) // 32
        self.k_off = torch.empty(nsl + 1, dtype=torch.int64, device=self.dev)
        elems = C.c_int64(0)
        _raise_for(self.h.L.vfpi_sell_layout_device(self.h.h, pile.n, self.k[0].data_ptr(), self.k_off.data_ptr(),
                                                    C.byref(elems)), self.h)
        self.k_val = torch.empty(max(elems.value, 1), dtype=torch.float64, device=self.dev)
        self.k_col = torch.empty(max(elems.value, 1), dtype=torch.int32, device=self.dev)
        _raise_for(self.h.L.vfpi_sell_pack_device(self.h.h, pile.n, self.k[0].data_ptr(), self.k[1].data_ptr(),
                                                  self.k[2].data_ptr(), self.k_off.data_ptr(),
                                                  self.k_val.data_ptr(), self.k_col.data_ptr()), self.h)
        self.k = None  # the CSR copy is no longer needed on the device
        self.m, self.g = up(pile.m, np.float64), up(pile.gravity, np.float64)
        self.X = up(pile.X.ravel(), np.float64)
        self.x = up(pile.x.ravel(), np.float64)
        self.v = up(pile.v.ravel(), np.float64)
        self.prev = None
        self.steps = 0
        self.geo_t = (up(pile.surf, np.int32), up(pile.tris.ravel(), np.int32), up(pile.node_body_i32(), np.int32),
                      up(pile.tri_cube, np.int32))
        g = _lib.VfpiPileGeometry()
        g.nodes, g.n_surf, g.n_tris = pile.n // 3, pile.surf.shape[0], pile.tris.shape[0]
        g.surf, g.tris, g.node_body, g.tri_body = (t.data_ptr() for t in self.geo_t)
        g.reach, g.cell, g.neg_half_h = max(0.5 * pile.h, pile.margin), 2.0 * pile.h, -0.5 * pile.h
        g.margin, g.mu = pile.margin, pile.mu
        g.neg_beta_dt, g.e_rest, g.rest_threshold = -(pile.beta / pile.dt), pile.e_rest, pile.thr
        self.geo = g

    def state(self):
        """(x, v) of the device state as host arrays (n_nodes, 3)."""
        return self.x.cpu().numpy().reshape(-1, 3), self.v.cpu().numpy().reshape(-1, 3)

    def device_contacts(self) -> PileContacts:
        """Device detection + nodalization of the current device state, copied
        to the host (for checks; the step keeps them on the device)."""
        import ctypes as C

        import torch

        from . import _lib
        from .solver import _raise_for

        h = self.h
        oc = _lib.VfpiPileContacts()
        st = torch.cuda.current_stream(self.device)
        sp_ = C.c_void_p(st.cuda_stream if st.cuda_stream else 1)
        _raise_for(h.L.vfpi_pile_contacts_device(h.h, C.byref(self.geo), self._p(self.x), self._p(self.v),
                                                 C.byref(oc), sp_), h)
        st.synchronize()
        n_c, nv3, nj = int(oc.n_c), 3 * int(oc.n_virtual), int(oc.jv_nnz)

        def d2h(p, n, dt):
            t = torch.empty(n, dtype=dt, device=self.dev)
            if n:
                torch.cuda.synchronize(self.device)
                _lib_cuda_copy(t, p, n, dt)
            return t.cpu().numpy()

        i32, f64 = torch.int32, torch.float64
        ci, cj = d2h(oc.col_i, n_c, i32), d2h(oc.col_j, n_c, i32)
        fr, mu, phi = d2h(oc.frames, 9 * n_c, f64), d2h(oc.mu, n_c, f64), d2h(oc.phi, n_c, f64)
        jp, ji, jx = d2h(oc.jv_indptr, nv3 + 1, i32), d2h(oc.jv_indices, nj, i32), d2h(oc.jv_data, nj, f64)
        jv = sp.csr_matrix((jx, ji, jp), shape=(nv3, self.pile.n))
        return PileContacts(ci.astype(np.int64), cj.astype(np.int64), fr.reshape(-1, 3, 3), phi, mu, jv,
                            int(oc.n_ground), int(oc.n_face))

    def _p(self, t):
        import ctypes as C

        return C.c_void_p(t.data_ptr())

    def step(self, cfg) -> dict:
        import ctypes as C
        import time

        import torch

        from . import _lib
        from ._lib import VfpiAugmented, VfpiAugmentInput, VfpiResult, VfpiSystem
        from .solver import _c_config, _raise_for

        pile, h, dev, P = self.pile, self.h, self.dev, self._p
        st = torch.cuda.current_stream(self.device)
        sp_ = C.c_void_p(st.cuda_stream if st.cuda_stream else 1)
        t0 = time.perf_counter()
        n_o = pile.n
        zmin = self.x.view(-1, 3)[:, 2].min()  # read after the step's final sync (no extra round trip)
        i32, f64 = _lib._i32p, _lib._f64p
        oc = _lib.VfpiPileContacts()
        _raise_for(h.L.vfpi_pile_contacts_device(h.h, C.byref(self.geo), P(self.x), P(self.v), C.byref(oc), sp_), h)
        n_c, nv3, jnnz = int(oc.n_c), 3 * int(oc.n_virtual), int(oc.jv_nnz)
        counts = dict(n_ground=int(oc.n_ground), n_face=int(oc.n_face), n_virtual=int(oc.n_virtual))
        jp_, ji_, jx_ = oc.jv_indptr, oc.jv_indices, oc.jv_data
        cptr = (oc.col_i, oc.col_j, oc.frames, oc.mu, oc.phi)
        t_detect = time.perf_counter() - t0
        n = n_o + nv3
        b = torch.zeros(n, dtype=torch.float64, device=dev)
        _raise_for(h.L.vfpi_fem_rhs_sell_device(h.h, n_o, P(self.k_off), P(self.k_val), P(self.k_col), P(self.x),
                                                P(self.X), P(self.v), P(self.m), P(self.g), pile.dt, P(b), sp_), h)
        inp = VfpiAugmentInput(n_o, nv3, int(pile.a_data.shape[0]), C.cast(P(self.a[0]), i32),
                               C.cast(P(self.a[1]), i32), C.cast(P(self.a[2]), f64), jnnz, jp_, ji_, jx_,
                               float(pile.k_v))
        out = VfpiAugmented()
        _raise_for(h.L.vfpi_augment_device(h.h, C.byref(inp), C.byref(out), sp_), h)
        warm = torch.zeros(n, dtype=torch.float64, device=dev)
        if self.prev is not None:
            warm[:n_o] = self.prev
            if nv3:
                vp = C.c_void_p
                _raise_for(h.L.vfpi_csr_matvec_device(h.h, nv3, C.cast(jp_, vp), C.cast(ji_, vp), C.cast(jx_, vp),
                                                      P(warm), P(warm[n_o:]), sp_), h)
        s = VfpiSystem()
        s.n, s.n_c, s.nnz = n, n_c, int(out.nnz)
        s.indptr, s.indices, s.data = out.indptr, out.indices, out.data
        s.b = C.cast(P(b), f64)
        s.col_i, s.col_j, s.frames, s.mu, s.phi = cptr
        s.mu2 = cptr[3]
        vh = torch.empty(n, dtype=torch.float64, device=dev)
        lam = torch.empty(max(3 * n_c, 1), dtype=torch.float64, device=dev)
        trace = torch.empty(max(cfg.max_iters, 1), dtype=torch.float64, device=dev)
        res = VfpiResult()
        res.v, res.lam, res.residual_trace = (C.cast(P(t), _lib._f64p) for t in (vh, lam, trace))
        res.scc, res.w = None, None
        code = h.L.vfpi_solve_device(h.h, C.byref(s), _c_config(cfg), C.cast(P(warm), _lib._f64p), None, C.byref(res),
                                     sp_)
        _raise_for(code, h)
        code = h.L.vfpi_wait(h.h, C.byref(res))
        if code not in (_lib.OK, _lib.DIVERGED):
            _raise_for(code, h)
        diverged = code == _lib.DIVERGED
        if diverged:
            # the reference's flagged contact-free step (harness.py:586-593):
            # v_hat = cg(A_o, b_o, rtol=1e-10, maxiter=10 n_o), virtual rows 0, lam = 0
            cg_it = C.c_int32(0)
            _raise_for(h.L.vfpi_cg_device(h.h, n_o, P(self.a[0]), P(self.a[1]), P(self.a[2]), P(b), P(vh), 1e-10,
                                          10 * n_o, C.byref(cg_it), sp_), h)
            vh[n_o:] = 0.0
            lam.zero_()
        _raise_for(h.L.vfpi_advance_device(h.h, n_o, pile.dt, P(vh), P(self.x), P(self.v), sp_), h)
        self.prev = vh[:n_o].clone()
        it = int(res.iterations)
        scalars = torch.stack([zmin, 0.5 * torch.dot(self.m * self.v, self.v),
                               trace[it - 1] if it > 0 and not diverged else
                               torch.zeros((), dtype=torch.float64, device=dev)])
        zmin_h, ke, resid = scalars.tolist()  # the step's one closing synchronisation
        max_pen = max(0.0, -zmin_h)
        self.steps += 1
        self.last = dict(v_hat=vh, lam=lam[: 3 * n_c])
        # a diverged step reports iters 0 / residual 0 like the harness row
        # (harness.py:549-553, the exception skips their assignment);
        # vfpi_iterations is the V-FPI work the device did either way
        return dict(n_c=n_c, **counts, n=n, nnz=int(out.nnz), vfpi_iterations=it,
                    iterations=0 if diverged else it, converged=bool(res.converged) and not diverged,
                    diverged=diverged,
                    setup_ms=float(res.setup_ms), loop_ms=float(res.loop_ms), detect_s=t_detect,
                    residual=resid, max_pen_m=max_pen, ke_J=ke,
                    wall_s=time.perf_counter() - t0)

    def metrics_row(self, step: int, r: dict):
        """``harness.MetricsRow`` of one step result (``harness.py:598-611``):
        dyn_ms = detection + nodalization, solve_ms = setup + loop, ke_J of the
        integrated state, max_pen_m = deepest plane penetration at the start of
        the step (face-contact depths are not included)."""
        return step_metrics_row(step, r)


def step_metrics_row(step: int, r: dict):
    """``harness.MetricsRow`` (``harness.py:598-611``) of a ``PileStepper.step`` result."""
    from .metrics import MetricsRow

    return MetricsRow(step=step, dyn_ms=1e3 * r["detect_s"], solve_ms=r["setup_ms"] + r["loop_ms"],
                      iters=r["iterations"], residual=r["residual"], max_pen_m=r["max_pen_m"], contacts=r["n_c"],
                      ke_J=r["ke_J"], diverged=r["diverged"], converged=r["converged"])


def run_piles_sharded(n_scenes: int, steps: int, cfg, make_pile, stepper=None, group=None, keep_rows=True):
    """configs[4] scene variants sharded over ranks: every rank
    builds and steps its contiguous block of scenes (``batch.shard_bounds``)
    with no data-path collective; at the end the counters are sum-reduced, the
    wall time max-reduced, and rank 0 gathers every scene's final (x, v) and
    per-step rows in scene order.

    ``make_pile(scene) -> CubePile``; ``stepper(pile) -> obj`` with
    ``.step(cfg) -> dict`` and ``.state() -> (x, v)`` (default: ``PileStepper``
    on the current CUDA device). Returns (per-scene results on rank 0 else
    None, totals)."""
    import time

    import torch
    import torch.distributed as dist

    from .batch import shard_bounds

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    lo, hi = shard_bounds(n_scenes, world, rank)
    if stepper is None:
        stepper = lambda p: PileStepper(p, device=torch.cuda.current_device())  # noqa: E731
    local, ci, its, nsteps = [], 0, 0, 0
    build_s = 0.0
    t0 = time.perf_counter()
    for sc in range(lo, hi):
        tb = time.perf_counter()
        st = stepper(make_pile(sc))
        build_s += time.perf_counter() - tb
        rows = []
        for _ in range(steps):
            r = st.step(cfg)
            ci += r["n_c"] * r.get("vfpi_iterations", r["iterations"])
            its += r.get("vfpi_iterations", r["iterations"])
            nsteps += 1
            if keep_rows:
                rows.append(dict(r))
        x, v = st.state()
        local.append(dict(scene=sc, x=np.asarray(x), v=np.asarray(v), rows=rows))
    wall = time.perf_counter() - t0 - build_s
    totals = {"contact_iterations": ci, "iterations": its, "scene_steps": nsteps, "wall_s": wall}
    if world == 1:
        return local, totals
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else None
    t = torch.tensor([float(ci), float(its), float(nsteps)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    w = torch.tensor([wall], dtype=torch.float64, device=dev)
    dist.all_reduce(w, op=dist.ReduceOp.MAX, group=group)
    totals = {"contact_iterations": int(t[0].item()), "iterations": int(t[1].item()), "scene_steps": int(t[2].item()),
              "wall_s": float(w[0].item())}
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(local, gathered, dst=0, group=group)
    if rank != 0:
        return None, totals
    return [s for part in gathered for s in part], totals
