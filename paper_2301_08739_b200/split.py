"""Group-range split of ONE large scene across ranks (BASELINE config 4).

Every rank holds the replicated coordinates and builds the identical index schedule
(`fwa_b200_split_begin`).  Block b's window-sort order is cut into P contiguous ranges of
whole groups; rank r computes its range (`fwa_b200_split_block`), the ranks all-gather
the sorted-order output rows (NCCL over NVLink on GPUs), and every rank scatters them back
to pillar-id order (`fwa_b200_split_scatter`) because block b+1 re-sorts with another
(axis, shift) and needs rows from everywhere (flatten.hpp:150-161, backbone.hpp:215-317).

`split_forward` is written against a small runner interface so the identical host logic
runs on the GPU (`DeviceRunner`, the C ABI) and in the CPU gloo tests (an oracle runner).
"""
from __future__ import annotations

import math
from typing import Callable, List, Tuple


def partition_groups(n_groups: int, world: int) -> Tuple[List[Tuple[int, int]], int]:
    """Contiguous equal chunks of groups (the last rank may hold fewer): returns the
    per-rank [g0, g1) ranges and the chunk size used to pad the all-gather."""
    per = max(1, math.ceil(n_groups / world))
    ranges = [(min(r * per, n_groups), min((r + 1) * per, n_groups)) for r in range(world)]
    return ranges, per


def split_forward(runner, n_blocks: int, group_size: int, world: int, rank: int,
                  all_gather: Callable, alloc: Callable):
    """runner: begin() -> K;  block(b, g0, g1, x, y_local);  scatter(b, y_all, dst);
    input() -> block 0's input rows; x_buffer(), out_buffer() -> buffers.
    all_gather(dst, src): rank-ordered concatenation of equal-size chunks.
    alloc(rows) -> a rows x D buffer.  Returns the runner's output buffer."""
    K = runner.begin()
    n_groups = K // group_size
    ranges, per = partition_groups(n_groups, world)
    g0, g1 = ranges[rank]
    y_local = alloc(per * group_size)
    y_all = alloc(world * per * group_size)
    x = runner.input()
    for b in range(n_blocks):
        runner.block(b, g0, g1, x, y_local)
        all_gather(y_all, y_local)  # rank r's chunk starts at group r*per: concat == sorted order
        dst = runner.out_buffer() if b == n_blocks - 1 else runner.x_buffer()
        runner.scatter(b, y_all, dst)
        x = dst
    return runner.out_buffer()


class DeviceRunner:
    """The C-ABI implementation (torch tensors for device memory)."""

    def __init__(self, ctx, d_coords, d_feats, cfg):
        import torch
        self.ctx, self.cfg = ctx, cfg
        self.d_coords, self.d_feats = d_coords, d_feats
        self.n = d_coords.shape[0]
        dev = d_feats.device
        self.x = torch.empty((self.n, cfg.d_model), dtype=torch.float32, device=dev)
        self.out = None
        self.dev = dev

    def begin(self):
        import torch
        K = self.ctx.split_begin(self.d_coords.data_ptr(), self.n, self.cfg)
        self.out = torch.empty((K, self.cfg.d_model), dtype=torch.float32, device=self.dev)
        return K

    def input(self):
        return self.d_feats

    def x_buffer(self):
        return self.x

    def out_buffer(self):
        return self.out

    def block(self, b, g0, g1, x, y_local):
        self.ctx.split_block(b, g0, g1, x.data_ptr(), y_local.data_ptr())

    def scatter(self, b, y_all, dst):
        self.ctx.split_scatter(b, y_all.data_ptr(), dst.data_ptr())
