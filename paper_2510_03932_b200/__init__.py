"""octgpu: B200-native (sm_100a) evaluation hot path of the arXiv 2510.03932
reference (`octrans`): per-node fp64 objective / constraint / gradient /
Jacobian / Lagrangian-Hessian evaluation into the reference's COO slots, the
atomic-free KKT assembly and the interior-point vector kernels, behind the
reference's EvalContext / KktAssembler interface (include/octgpu.h).
"""
from .evaluation import (BandLdl, Comm, EvalContext, KktAssembler, Model, Solver, objective_chunk_owners, ref_symbolic,  # noqa: F401
                         shard_plan, solve, solve_batch, synth_uniform)
from .models import MODELS  # noqa: F401

__all__ = ["BandLdl", "Comm", "shard_plan", "ref_symbolic", "EvalContext", "KktAssembler", "Model", "MODELS", "Solver", "objective_chunk_owners", "solve", "solve_batch",
           "synth_uniform"]
