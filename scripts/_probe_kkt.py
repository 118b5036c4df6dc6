"""Probe: the reference's first Goddard KKT (REF_DUMP_KKT) factored by the device band LDL^T at several (dw, dc)."""
import os, sys
import numpy as np, scipy.io as sio, scipy.sparse as sp, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
os.environ["REF_DUMP_KKT"] = "/tmp/g_kkt.mtx"
from _oracle import RefModel
from paper_2510_03932_b200 import MODELS, Model, EvalContext, KktAssembler, BandLdl
from paper_2510_03932_b200.evaluation import LIB, _cuda_memcpy_d2d, _ptr
N = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
RefModel(MODELS['goddard'], N).solve(parallel=False, max_iter=1)
del os.environ["REF_DUMP_KKT"]
A = sp.tril(sio.mmread('/tmp/g_kkt.mtx')).tocsc()
A.sort_indices()
m = Model(MODELS['goddard'], N); ec = EvalContext(m); k = KktAssembler(m, ec)
colp, rowi = k.pattern()
assert np.array_equal(colp, A.indptr) and np.array_equal(rowi, A.indices), "pattern mismatch"
vals = torch.tensor(A.data, dtype=torch.float64, device='cuda')
for seg in (None, "1"):
    if seg: os.environ["OCG_LDL_SEGMENTS"] = seg
    k.assemble(np.ones(k.ntot))  # then overwrite
    torch.cuda.synchronize()
    _cuda_memcpy_d2d(LIB.ocg_kkt_values(k._h), _ptr(vals), vals.numel() * 8)
    ldl = BandLdl(k)
    print("segments", seg, ldl.info())
    for dw, dc in [(0, 0), (1e-4, 0), (1e-4, 1e-8 * 0.1 ** 0.25), (3.3e-5, 0)]:
        print("  dw", dw, "dc", dc, "inertia", ldl.factor(dw, dc), "expect", (k.ntot, k.dim - k.ntot, 0))
