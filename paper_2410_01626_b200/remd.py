"""pH replica exchange across contexts / GPUs.

One attempt: every rank's context writes its (label, E_0..E_{P-1}) rows into a device
tensor (cph_exchange_energies), one all-gather over the process group (NCCL over
NVLink/NVSwitch on GPUs) concatenates them in rank order, and every rank applies the same
Metropolis decisions to its own replicas (cph_exchange_apply).  Nothing goes through the
host: the gather and the library kernels are ordered on the current CUDA stream.

Layout contract: every rank holds the same number R of replicas, created with
remd_first = rank * R and remd_total = world * R; ladders are consecutive blocks of P
global replicas.  Argument marshalling only - the decisions run in libcph.so.
"""
from __future__ import annotations


def exchange_step(ctx, seed: int, attempt: int, group=None):
    """Attempt one round of neighbour swaps (pairs p = attempt % 2, +2, ...)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    width = ctx.R * (ctx.P + 1)
    device = ctx.exchange_device()
    local = torch.empty(width, dtype=torch.float64, device=device)
    ctx.exchange_energies_into(local)
    if world == 1:
        ctx.exchange_apply_from(local, seed, attempt)
        return
    gathered = torch.empty(world * width, dtype=torch.float64, device=device)
    dist.all_gather_into_tensor(gathered, local, group=group)
    ctx.exchange_apply_from(gathered, seed, attempt)


def run(ctx, n_steps: int, stride: int, seed: int, first_attempt: int = 0, group=None) -> int:
    """Alternate cph_step(stride) and one exchange attempt until n_steps are done; returns
    the next attempt index."""
    attempt = first_attempt
    done = 0
    while done < n_steps:
        k = min(stride, n_steps - done)
        ctx.cph_step(k)
        done += k
        if k == stride:
            exchange_step(ctx, seed, attempt, group)
            attempt += 1
    return attempt
