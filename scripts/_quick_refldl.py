import sys, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from _oracle import RefEval, RefKkt, RefModel
from paper_2510_03932_b200 import MODELS, BandLdl, EvalContext, KktAssembler, Model
for name, N in [("double_integrator", 200), ("goddard", 1000)]:
    m, r = Model(MODELS[name], N), RefModel(MODELS[name], N)
    ec, re = EvalContext(m), RefEval(r)
    x, lam = r.synth_acceptance(20250808)
    c = torch.empty(m.m_con, dtype=torch.float64, device=ec.device)
    ec.eval_constraints_jacobian(x, c); ec.eval_hessian(x, lam)
    re.constraints_jacobian(x); re.hessian(x, lam)
    k, kr = KktAssembler(m, ec), RefKkt(re)
    k.assemble(np.random.default_rng(5).uniform(0.5, 2.0, k.ntot))
    val = k.values().cpu().numpy()
    ldl = BandLdl(k, order="reference")
    print(name, "factor", ldl.factor(1e-4, 1e-8), flush=True)
    b = np.random.default_rng(9).standard_normal(k.dim)
    xs = ldl.solve(b).cpu().numpy()
    torch.cuda.synchronize()
    xr = kr.factor_solve(val, b, 1e-4, 1e-8)
    print(name, "solve rel", np.max(np.abs(xs - xr)) / np.max(np.abs(xr)), flush=True)
