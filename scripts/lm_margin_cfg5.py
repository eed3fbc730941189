import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle as O, pget_data as P, paper_2604_26745_b200 as pg
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.float32)).cuda()
cid = 5; cfg = P.CONFIGS[cid]; gd = P.geometry_desc(cid); B = gd["batch"]
g = pg.Geometry(gd); g1 = dict(gd, batch=1)
lt, mt = P.make_phantom(cid)
ys = [P.poisson_noise(O.forward(g1, lt[k:k + 1], mt[k:k + 1]), 1e4, 50 + k) for k in range(4)]
y = np.concatenate([ys[m % 4] for m in range(B)])
l0, m0 = P.initial_guess(gd["n_px"], B)
sl, sm, st = pg.gn_cg_step(g, dev(l0), dev(m0), dev(y), cfg.alpha, 0.0, cfg.n_cg)
torch.cuda.synchronize()
S = pg.read_stats(st, B, cfg.n_cg)
for m in (1, 38):
    k = m % 4
    _, _, So = O.gn_cg_step(g1, l0[m:m + 1], m0[m:m + 1], ys[k], cfg.alpha, 0.0, cfg.n_cg)
    print(m, "pred rel", abs(S[m]["pred"] - So["pred"]) / abs(So["pred"]), "rho abs", abs(S[m]["rho"] - So["rho"]),
          "cg_res1 rel", abs(S[m]["cg_res"][1] - So["cg_res"][1]) / So["cg_res"][1], flush=True)
preds = np.array([S[m]["pred"] for m in range(B)])
print("pred spread over identical problems (m % 4 == 2):", np.ptp(preds[2::4]) / np.mean(preds[2::4]))
