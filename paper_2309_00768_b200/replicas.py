"""Multi-GPU policy: replicas only.

The exact sequential time sweeps of P_T (precond.py:122-131, 194-205) do not
shard across devices, so N GPUs run N independent space-time solves (one
process per GPU).  Throughput is aggregated the way the benchmark contract
requires: total work of all ranks over the max-over-ranks device time.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def aggregate(seconds: float, work: float, device=None) -> tuple[float, float]:
    """(max seconds over ranks, summed work over ranks); identity when not
    running distributed.  Works on the gloo (CPU) and nccl (GPU) backends."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(seconds), float(work)
    dev = device if device is not None else torch.device("cpu")
    t = torch.tensor([float(seconds)], dtype=torch.float64, device=dev)
    w = torch.tensor([float(work)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(w, op=dist.ReduceOp.SUM)
    return float(t), float(w)
