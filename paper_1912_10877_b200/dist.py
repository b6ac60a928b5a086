"""Multi-GPU execution over torch.distributed.

* Batched registers (the QCBM configuration): the batch shards across ranks; forward, seed and
  reverse pass are rank-local on each rank's B-shard (batch-innermost registers); then ONE
  all-reduce(sum) of the P-vector of parameter gradients (gradients sum over the
  batch) and an all-gather of the per-batch energies.  This is the only real exchange of the
  path.  Gradients are summed in rank order by the collective, so the result equals the
  single-GPU batched gradient up to the order of one P-length sum.
* The 25-qubit metric state fits one B200: `bench.py --gpus N` runs N replicas, no collective.

The per-rank compute is the device engine (`expect_grad`); `local_step` is injectable so the
collective logic can be tested with the gloo backend on CPU (tests/test_dist.py) against the
CPU oracle — the product path never computes on the CPU.
"""
from __future__ import annotations

from typing import Callable, Sequence

import numpy as np


def shard_range(nbatch: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous balanced split of [0, nbatch): the first nbatch % world ranks get one more."""
    base, extra = divmod(nbatch, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _device_step(obs, circuit, reg):
    from .ad import expect_grad
    r = expect_grad(obs, (reg, circuit))
    return r.energies, r.param_grads


def sharded_expect_grad(obs, circuit, local_reg, nbatch: int, group=None,
                        local_step: Callable | None = None) -> tuple[np.ndarray, np.ndarray]:
    """expect'(O, reg => circuit) for a batch sharded over the ranks of `group`.

    `local_reg` holds this rank's shard (rows shard_range(nbatch, rank, world)).  Returns the
    full per-batch energies (all ranks) and the batch-summed gradient (identical on all ranks).
    """
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    step = local_step or _device_step
    e_local, g_local = step(obs, circuit, local_reg)
    e_local = np.asarray(e_local, dtype=np.float64)
    g_local = np.asarray(g_local, dtype=np.float64)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else torch.device("cpu")
    g = torch.from_numpy(g_local.copy()).to(dev)
    dist.all_reduce(g, op=dist.ReduceOp.SUM, group=group)
    # energies: shards are contiguous and balanced, pad to the largest shard and gather
    sizes = [shard_range(nbatch, r, world)[1] - shard_range(nbatch, r, world)[0] for r in range(world)]
    mx = max(sizes)
    pad = torch.zeros(mx, dtype=torch.float64, device=dev)
    pad[: e_local.size] = torch.from_numpy(e_local).to(dev)
    outs = [torch.zeros(mx, dtype=torch.float64, device=dev) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    energies = np.concatenate([o.cpu().numpy()[: sizes[r]] for r, o in enumerate(outs)])
    return energies, g.cpu().numpy()


def product_batch(nqubits: int, nbatch: int, seed: int = 42) -> list[int]:
    """QCBM inputs (SURVEY §8(d) cfg 3): basis states Rng(seed).bits() & (2^n - 1), one per batch."""
    from .register import Rng
    r = Rng(seed)
    mask = (1 << nqubits) - 1
    return [r.bits() & mask for _ in range(nbatch)]


def batch_of(bits: Sequence[int], lo: int, hi: int) -> list[int]:
    return list(bits[lo:hi])
