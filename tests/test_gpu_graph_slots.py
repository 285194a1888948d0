"""Setup-graph cache with two slots (vfpi_api.cu SetupGraphSet): a caller that
alternates two device input buffers gets both setups captured and replayed,
and every solve still matches the oracle bit for bit."""

import numpy as np
import pytest
import torch

from paper_2201_09212_b200 import _lib
from paper_2201_09212_b200.device import DeviceSystem
from paper_2201_09212_b200.scenes import rigid_contact_system
from paper_2201_09212_b200.solver import SolverConfig


@pytest.mark.gpu
def test_alternating_input_buffers_replay_both_graphs():
    from oracle import vfpi_oracle as O

    ps = rigid_contact_system(n_bodies=96, n_contacts=320, seed=4)
    cfg = SolverConfig(residual_tol=1e-8, max_iters=40)
    s = O.System(ps.n, ps.indptr, ps.indices, ps.data, ps.b, ps.col_i.astype(np.int64), ps.col_j.astype(np.int64),
                 ps.frames.reshape(-1, 3, 3), ps.mu, ps.mu2, ps.phi)
    vo, lo, ro = O.solve(s, O.Config(residual_tol=1e-8, max_iters=40), np.zeros(ps.n))
    st = torch.cuda.Stream()
    bufs = [DeviceSystem(ps, 0), DeviceSystem(ps, 0)]
    warm = torch.zeros(ps.n, dtype=torch.float64, device="cuda")
    h = _lib.handle(0)
    launches = []
    for k in range(8):
        ds = bufs[k % 2]
        before = h.launches()
        with torch.cuda.stream(st):
            ds.enqueue(cfg, warm, st)
            res = ds.finish()
        launches.append(h.launches() - before)
        assert res.iterations == ro.iterations
        assert np.array_equal(ds.v.cpu().numpy()[: ps.n], vo), k
        assert np.array_equal(ds.lam.cpu().numpy()[: 3 * ps.n_c].reshape(-1, 3), lo), k
    # eager, eager, capture, capture, then replays: the last calls launch as few kernels as the replays
    assert launches[-1] == launches[-2] == launches[-3]
