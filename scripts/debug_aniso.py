"""Debug: strict-anisotropic one-shot GPU vs oracle on random inputs with mu2 != mu."""
import sys
sys.path.insert(0, ".")
import numpy as np
from oracle import vfpi_oracle as O
from paper_2201_09212_b200 import solver as S
g = np.random.default_rng(1)
n = 4000
eta = g.standard_normal((n, 3)) * 3
gam = g.uniform(0.5, 2, n)
phi = g.uniform(-1, 0, n)
mu = g.uniform(0.2, 0.8, n)
mu2 = g.uniform(0.1, 0.9, n)
lo = O.oneshot(gam, eta, phi, mu, mu2, "strict-anisotropic")
lg = S.contact_solve_oneshot(S.SurrogateDelassus(gam), eta, phi, mu, "strict-anisotropic", mu2)
d = np.abs(lg - lo).max(axis=1)
bad = np.nonzero(d > 0)[0]
print("mismatch", bad.size, "of", n, "max", d.max())
for k in bad[:5]:
    print(k, "eta", eta[k], "gam", gam[k], "phi", phi[k], "mu", mu[k], "mu2", mu2[k])
    print("   gpu", lg[k], "\n   ora", lo[k])
