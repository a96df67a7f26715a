"""Multi-GPU partitioning of the TN-linear forward (one process per GPU).

Three ways to spread the work:

* replicas      — independent decode streams: every rank holds the whole
                  (small) TN layer and serves its own tokens. No collective.
* token-sharded — prefill: rank g takes tokens [g*M/G, (g+1)*M/G). No collective.
* output-sharded — prefill with one exchange step: rank g owns the output rows
                  of its slice of the leading output mode i0 (the row range is
                  contiguous because row modes come first,
                  tn_decompositions.py:59-63) and computes only those; the
                  input side up to the cut is recomputed on every rank (r_cut
                  per token). Its kernels store the slice straight into its
                  columns of the token-major y (a strided TMA store, no staging).
                  Exchange, NCCL groups: y lives in symmetric memory and every
                  rank writes its slice into the same columns of every peer's y
                  over NVLink (P2P stores), then one device-side barrier — the
                  only traffic beyond the local store is the (G-1)/G * M * rows
                  NVLink ingress, and there is no gather buffer and no permute.
                  Other backends (gloo in the CPU tests) all-gather the slices
                  into [G][M][rows/G] and place them.

The local compute is the C-ABI forward of a row-restricted plan
(``tnl_plan_create_rows``). For CPU tests the compute callable can be
injected (the gloo tests pass the oracle); the product path has no CPU
compute.
"""

from __future__ import annotations

import math
from typing import Callable

import torch
import torch.distributed as dist

from .errors import ShapeError
from .layer import CompressedLayer


def output_shard_ranges(mode_shape, row_mode_count: int, world: int) -> list[tuple[int, int]]:
    """Row range per rank: slices of the leading output mode i0 when it divides,
    else equal contiguous row blocks (rows must then divide by world)."""
    ms = tuple(mode_shape)
    rows = math.prod(ms[:row_mode_count])
    n0 = ms[0]
    if n0 % world == 0:
        per = rows // world  # = (n0 / world) * prod(ms[1:rm])
    elif rows % world == 0:
        per = rows // world
    else:
        raise ShapeError(f"{rows} output rows (leading mode {n0}) cannot be split over {world} ranks")
    return [(g * per, (g + 1) * per) for g in range(world)]


def token_shard_range(m: int, rank: int, world: int) -> tuple[int, int]:
    per = (m + world - 1) // world
    lo = min(m, rank * per)
    return lo, min(m, lo + per)


class OutputShardedLayer:
    """Output-mode-sharded forward with one exchange step (prefill / large M).

    exchange: "auto" (symmetric-memory P2P on NCCL groups, else all-gather), "p2p", "allgather".
    The P2P path returns its own symmetric buffer (valid until the next forward on this layer);
    pass ``out`` to get a copy instead."""

    def __init__(self, layer: CompressedLayer, group=None, dtype=torch.bfloat16, device=None,
                 local_forward: Callable | None = None, exchange: str = "auto"):
        self.layer = layer
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.ranges = output_shard_ranges(layer.mode_shape, layer.row_mode_count, self.world)
        self.row_range = self.ranges[self.rank]
        self.rows, self.cols = layer.matrix_shape
        self.dtype = dtype
        if local_forward is None:
            plan = layer.plan(dtype, device, row_range=self.row_range)
            local_forward = plan.forward
        self.local_forward = local_forward
        if exchange not in ("auto", "p2p", "allgather"):
            raise ValueError(f"exchange must be auto / p2p / allgather, got {exchange!r}")
        self.exchange = exchange
        self._symm = None  # (m, device, buffer, handle)

    def _use_p2p(self, device) -> bool:
        if self.exchange == "allgather" or device.type != "cuda":
            return False
        try:
            nccl = dist.get_backend(self.group) == "nccl"
        except Exception:
            nccl = False
        if not nccl:
            if self.exchange == "p2p":
                raise ShapeError("exchange='p2p' needs an NCCL process group")
            return False
        return True

    def _symm_buffer(self, m: int, device):
        if self._symm is None or self._symm[0] != m or self._symm[1] != device:
            import torch.distributed._symmetric_memory as symm_mem

            buf = symm_mem.empty((m, self.rows), dtype=self.dtype, device=device)
            hdl = symm_mem.rendezvous(buf, self.group if self.group is not None else dist.group.WORLD)
            self._symm = (m, device, buf, hdl)
        return self._symm[2], self._symm[3]

    def forward(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        m = x.shape[0]
        lo, hi = self.row_range
        per = hi - lo
        if self._use_p2p(x.device):
            y, hdl = self._symm_buffer(m, x.device)
            hdl.barrier(channel=0)  # every rank is done with the previous result in its y
            self.local_forward(x, out=y[:, lo:hi])  # this rank's columns, stored in place
            for p in range(self.world):
                if p != self.rank:  # P2P stores of exactly this slice into the peer's y
                    hdl.get_buffer(p, (m, self.rows), self.dtype)[:, lo:hi].copy_(y[:, lo:hi])
            hdl.barrier(channel=1)  # every peer's slice has landed in our y
            if out is not None:
                out.copy_(y)
                return out
            return y
        # all-gather: this rank's rows go straight into its slot of the gather buffer, the gather
        # runs in place (input = output slot `rank`), then the slots are placed into y's columns
        flat = torch.empty((self.world * m, per), dtype=self.dtype, device=x.device)
        gathered = flat.view(self.world, m, per)
        try:
            self.local_forward(x, out=gathered[self.rank])
        except TypeError:  # injected compute without an `out` argument (CPU tests)
            y_local = self.local_forward(x)
            flat = torch.empty((self.world * m, per), dtype=y_local.dtype, device=y_local.device)
            gathered = flat.view(self.world, m, per)
            gathered[self.rank].copy_(y_local)
        dist.all_gather_into_tensor(flat, gathered[self.rank], group=self.group)
        y = out if out is not None else torch.empty((m, self.rows), dtype=flat.dtype, device=flat.device)
        y.view(m, self.world, per).copy_(gathered.permute(1, 0, 2))
        return y

    __call__ = forward


class TokenShardedLayer:
    """Token-sharded forward: rank g computes its own token block; no collective
    (``gather=True`` all-gathers the blocks, for checking)."""

    def __init__(self, layer: CompressedLayer, group=None, dtype=torch.bfloat16, device=None,
                 local_forward: Callable | None = None):
        self.layer = layer
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if local_forward is None:
            local_forward = layer.plan(dtype, device).forward
        self.local_forward = local_forward

    def forward(self, x_full: torch.Tensor, gather: bool = False) -> torch.Tensor:
        m = x_full.shape[0]
        if m % self.world and gather:
            raise ShapeError("gather=True needs M divisible by the world size")
        lo, hi = token_shard_range(m, self.rank, self.world)
        y = self.local_forward(x_full[lo:hi])
        if not gather:
            return y
        parts = torch.empty((self.world * y.shape[0],) + tuple(y.shape[1:]), dtype=y.dtype, device=y.device)
        dist.all_gather_into_tensor(parts, y.contiguous(), group=self.group)
        return parts

    __call__ = forward
