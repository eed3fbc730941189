"""CG sensitivity study behind the LM-iteration parity reading (R-LM).

Runs the config-2 GN-CG step (20 CG steps, alpha = 1e-3, beta = 0) with the fp64 oracle's H
operator, once exactly and twice with every H p perturbed by an independent relative N(0, 1e-7)
error (the size of an fp32 evaluation of H p), and reports how far s, pred = m(0) - m(s) and
f(u + s) move.  Calls only oracle/ (test infrastructure) and pget_data.  Output of the committed
run: profiles/cg_sensitivity_r01.txt.
"""
import sys, time; sys.path.insert(0,'.')
import numpy as np, oracle as O, pget_data as P
# usage: cg_sensitivity.py [cfg2 | cfg5:<member>] [eps ...]; cfg5:<m> is the problem of
# tests/test_gpu_parity.py::test_lm_iteration_config5_batched for batch member m
case = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
EPS = [float(x) for x in sys.argv[2:]] or [1e-7]
if case == "cfg2":
    cid=2; cfg=P.CONFIGS[cid]; gd=P.geometry_desc(cid)
    lt,mt=P.make_phantom(cid)
    y=P.poisson_noise(O.forward(gd,lt,mt),cfg.noise_peak,cfg.seed)
    l0,m0=P.initial_guess(gd['n_px'])
else:
    cid=5; cfg=P.CONFIGS[cid]; m=int(case.split(":")[1]); k=m%4
    gd=dict(P.geometry_desc(cid), batch=1)
    LT,MT=P.make_phantom(cid)
    lt,mt=LT[k:k+1],MT[k:k+1]
    y=P.poisson_noise(O.forward(gd,lt,mt),1e4,50+k)
    l0,m0=P.initial_guess(gd['n_px'])
t=time.time()
sl,sm,S=O.gn_cg_step(gd,l0,m0,y,cfg.alpha,0.0,cfg.n_cg)
print('oracle step',time.time()-t,'s; cg_res',S['cg_res'][[0,1,5,10,15,20]], 'pred',S['pred'],'rho',S['rho'])
s_ref=np.concatenate([sl.ravel(),sm.ravel()])
# reproduce CG in numpy with perturbed H
r=O.forward(gd,l0,m0)-y
gl,gm=O.vjp(gd,l0,m0,r.astype(np.float64))
Ll=O.laplacian(O.laplacian(l0)); Lm=O.laplacian(O.laplacian(m0))
b=-np.concatenate([(gl+cfg.alpha*Ll).ravel(),(gm+cfg.alpha*Lm).ravel()])
n=l0.size
def H(p):
    ql,qm=O.apply_H(gd,l0,m0,cfg.alpha,0.0,p[:n].reshape(l0.shape),p[n:].reshape(l0.shape))
    return np.concatenate([ql.ravel(),qm.ravel()])
def cg(eps,seed):
    rng=np.random.default_rng(seed)
    s=np.zeros_like(b); z=b.copy(); p=b.copy(); zeta=z@z
    for k in range(cfg.n_cg):
        q=H(p)
        if eps: q=q*(1+eps*rng.standard_normal(q.shape))
        g=p@q; a=zeta/g; s+=a*p; z-=a*q; z2=z@z; p=z+(z2/zeta)*p; zeta=z2
    return s
s0=cg(0,0); print('numpy CG vs oracle', np.linalg.norm(s0-s_ref)/np.linalg.norm(s_ref))
def pred_of(s):
    sl_,sm_=s[:n].reshape(l0.shape),s[n:].reshape(l0.shape)
    dy=O.jvp(gd,l0,m0,sl_,sm_)
    ls2=np.sum(O.laplacian(sl_)**2)+np.sum(O.laplacian(sm_)**2)
    return b@s-0.5*(np.sum(dy**2)+cfg.alpha*ls2)
def f_of(s):
    ul=l0+s[:n].reshape(l0.shape); um=m0+s[n:].reshape(l0.shape)
    r=O.forward(gd,ul,um)-y
    return 0.5*np.sum(r**2)+0.5*cfg.alpha*(np.sum(O.laplacian(ul)**2)+np.sum(O.laplacian(um)**2))
pr=pred_of(s_ref); fr=f_of(s_ref)
print('ref pred',pr,'f1',fr,'oracle',S['pred'],S['f_trial'])
for eps in EPS:
    for seed in [1,2,3]:
        s1=cg(eps,seed)
        print(case,'eps',eps,'seed',seed,'s diff',np.linalg.norm(s1-s_ref)/np.linalg.norm(s_ref),'pred rel',abs(pred_of(s1)-pr)/abs(pr),'f1 rel',abs(f_of(s1)-fr)/abs(fr), flush=True)
