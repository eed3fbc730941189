"""The README usage example, run as a script (checks that it stays runnable)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2604_26745_b200 as pg, pget_data as P
g = pg.Geometry(P.geometry_desc(2))
lam, mu = (torch.from_numpy(a).cuda() for a in P.make_phantom(2))
y = pg.forward(g, lam, mu)
s_lam, s_mu, stats = pg.gn_cg_step(g, lam, mu, y, alpha=1e-3, beta=0.0, n_cg=20)
m1, m2 = (torch.from_numpy(m).cuda() for m in P.prior_masks(2))
g.set_prior(m1, m2, alpha1=0.5, alpha2=2.0)
l0, m0 = (torch.from_numpy(a).cuda() for a in P.initial_guess(128))
per_iter = pg.lm_solve(g, l0, m0, y, n_iter=10, n_cg=20, alpha0=1e-2, k_freeze=3,
                       box=(0.0, 2.0, 0.0, 1.0), sgp=True, lam_per_mu=3.0)
print("readme example ok", per_iter[0][0]["f"], per_iter[-1][0]["f_trial"])
