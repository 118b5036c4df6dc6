"""Does the L2-flush kernel's shared-memory carveout cost the timed kernel?
Times the fused J+H launch (CUDA events) after the 512 MiB flush read, with
and without a small launch of a shared-memory-heavy kernel between the flush
and the start event (which leaves the SMs in the large-shared-memory
configuration)."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2510_03932_b200 import MODELS, EvalContext, Model  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream()
flush = torch.ones(bench.L2_FLUSH_BYTES // 8, dtype=torch.float64, device=dev)
sink = torch.zeros((), dtype=torch.float64, device=dev)
for name, N in [("goddard", 100_000), ("quadrotor", 100_000), ("hang_glider", 100_000)]:
    for block in (32, 128):
        m = Model(MODELS[name], N)
        x, lam = m.synth_acceptance(20250808)
        xd, ld = torch.as_tensor(x, device=dev), torch.as_tensor(lam, device=dev)
        c = torch.zeros(m.m_con, dtype=torch.float64, device=dev)
        ec = EvalContext(m, block=block)
        small = Model(MODELS[name], 64)
        xs, ls = (torch.as_tensor(a, device=dev) for a in small.synth_acceptance(1))
        cs = torch.zeros(small.m_con, dtype=torch.float64, device=dev)
        ecs = EvalContext(small, block=block)
        res = {}
        for mode in ("flush", "flush+small", "noflush"):
            ts = []
            for it in range(33):
                if mode != "noflush":
                    torch.sum(flush, dim=0, out=sink)
                if mode == "flush+small":
                    ecs.launch_jac_hess(xs, ls, cs, stream)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(stream)
                ec.launch_jac_hess(xd, ld, c, stream)
                e.record(stream)
                e.synchronize()
                ts.append(s.elapsed_time(e) * 1e3)
            res[mode] = float(np.median(ts[3:]))
        print(json.dumps({"model": name, "N": N, "block": block, **{k: round(v, 2) for k, v in res.items()}}), flush=True)
