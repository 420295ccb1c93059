"""Multi-GPU plumbing: row-slab partitions and the two collectives the path needs.

The reference is single-process; the only parallelism SURVEY.md §2.1/§8e
allows is row-slice data parallelism.  A rank owns a contiguous,
sigma-aligned slab of rows (so the implicit permutation stays rank-local and
the concatenation of slab packs equals the single-GPU pack).  Standalone SpMV
needs no collective (x replicated).  The PCG needs exactly two, over NCCL
(NVLink / NVSwitch) through torch.distributed:

* all-gather of the direction vector before every SpMV (in place: each rank's
  slab is its chunk of the global vector), and
* all-gather of the per-rank FP64 local dot sums, summed in rank order on the
  device (deterministic regardless of the collective's reduction tree).

`Comm` wraps a process group (NCCL on GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np


class Comm:
    """torch.distributed process-group wrapper used by the solvers and the bench."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        # NCCL moves device buffers directly over NVLink; gloo (CPU tests, or
        # several ranks sharing one GPU) stages through host memory
        self.nccl = dist.get_backend(group) == "nccl"

    def _gather(self, out_flat, local):
        if self.nccl or not out_flat.is_cuda:
            self.dist.all_gather_into_tensor(out_flat, local.contiguous(), group=self.group)
            return
        h_out = out_flat.cpu()
        self.dist.all_gather_into_tensor(h_out, local.contiguous().cpu(), group=self.group)
        out_flat.copy_(h_out)

    def all_gather_into(self, out_flat, local):
        """out_flat[r * len(local):(r+1) * len(local)] <- local of rank r (rank order)."""
        self._gather(out_flat, local)

    def all_gather_vec(self, full, local):
        """In-place all-gather of equal slabs: `local` is this rank's chunk of `full`."""
        if self.nccl or not full.is_cuda:
            self.dist.all_gather_into_tensor(full, local, group=self.group)
        else:
            self._gather(full, local.clone())

    def padded_len(self, n_glob: int) -> int:
        return n_glob

    def allreduce_max(self, v: int) -> int:
        import torch
        dev = "cuda" if torch.cuda.is_available() and self.dist.get_backend(self.group) == "nccl" else "cpu"
        t = torch.tensor([int(v)], dtype=torch.int64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return int(t.item())

    def barrier(self):
        self.dist.barrier(group=self.group)


def equal_row_slabs(n: int, world: int, sigma: int) -> List[Tuple[int, int]]:
    """sigma-aligned contiguous row slabs, as equal as the sigma granularity allows.

    The PCG requires exactly equal slabs (in-place all-gather of equal chunks),
    i.e. n % (world * sigma) == 0; `check_equal` enforces it.
    """
    nb = -(-n // sigma)
    out = []
    for r in range(world):
        a = min(n, (nb * r // world) * sigma)
        b = min(n, (nb * (r + 1) // world) * sigma)
        out.append((a, b))
    return out


def check_equal(slabs: Sequence[Tuple[int, int]]):
    sizes = {b - a for a, b in slabs}
    if len(sizes) != 1:
        raise ValueError(f"the distributed PCG needs equal row slabs, got sizes {sorted(sizes)}; "
                         "choose n divisible by world * sigma")


def word_balanced_slabs(row_words: np.ndarray, world: int, sigma: int) -> List[Tuple[int, int]]:
    """sigma-aligned slabs balancing stored words (power-law matrices).

    `row_words` are the per-row stored word counts (len + dummies, or the
    padded slice widths spread over rows); cuts are placed at sigma-block
    boundaries nearest to equal prefix sums.
    """
    n = len(row_words)
    nb = -(-n // sigma)
    blk = np.add.reduceat(np.asarray(row_words, dtype=np.int64), np.arange(0, n, sigma)) if n else np.zeros(0)
    pref = np.concatenate([[0], np.cumsum(blk)])
    total = pref[-1]
    cuts = [0]
    for r in range(1, world):
        target = total * r / world
        j = int(np.searchsorted(pref, target))
        j = min(max(j, cuts[-1]), nb)
        cuts.append(j)
    cuts.append(nb)
    return [(min(n, cuts[r] * sigma), min(n, cuts[r + 1] * sigma)) for r in range(world)]


def rank_order_sum(parts: np.ndarray) -> float:
    """Host mirror of psell_sum_strided: sequential sum in rank order."""
    s = 0.0
    for v in np.asarray(parts, dtype=np.float64):
        s += float(v)
    return s


__all__ = ["Comm", "equal_row_slabs", "check_equal", "word_balanced_slabs", "rank_order_sum"]
