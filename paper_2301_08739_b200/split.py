"""Group-range split of ONE large scene across ranks (BASELINE config 4).

Every rank holds the replicated coordinates and builds the identical index schedule
(`fwa_b200_split_begin`).  Block b's window-sort order is cut into P contiguous ranges of
whole groups; rank r computes its range (`fwa_b200_split_block`), the ranks all-gather
the sorted-order output rows (NCCL over NVLink on GPUs), and every rank scatters them back
to pillar-id order (`fwa_b200_split_scatter`) because block b+1 re-sorts with another
(axis, shift) and needs rows from everywhere (flatten.hpp:150-161, backbone.hpp:215-317).

`split_forward_a2a` replaces the all-gather between blocks by an all-to-all of only the
rows each rank needs for its next group range (the per-peer lists follow from the
replicated schedule), cutting the exchange from K rows to about K/P rows per rank.

`split_forward_p2p` fuses the exchange into the block kernel: rank r's block-b kernel
writes every output row straight into the x buffer of the rank whose block-(b+1) group range
holds that pillar (peer memory over NVLink: CUDA IPC mappings of the peers' buffers), and the
last block writes into rank 0's output -- no pack, no collective, no unpack; between blocks
the ranks only order themselves (`barrier`, e.g. a 1-element NCCL all-reduce on the stream).

`split_forward` is written against a small runner interface so the identical host logic
runs on the GPU (`DeviceRunner`, the C ABI) and in the CPU gloo tests (an oracle runner).
"""
from __future__ import annotations

import math
from typing import Callable, Optional, List, Tuple

import numpy as np


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


def exchange_tables(idx_b, idx_next, ranges, per, group_size, rank, world):
    """Block b -> b+1 exchange of `split_forward_a2a`: which of this rank's block-b output
    rows each peer needs for its block-(b+1) group range, and which pillar ids this rank
    receives from each peer.  Both sides list rows in the RECEIVER's block-(b+1) order, so
    the tables agree without communication (every rank holds the same schedule).
    Returns (send_local (concatenated local row indices), send_counts, recv_ids
    (concatenated pillar ids), recv_counts)."""
    import numpy as np
    idx_b = np.asarray(idx_b, np.int64)
    idx_next = np.asarray(idx_next, np.int64)
    chunk = per * group_size
    pos_b = np.empty(int(max(idx_b.max(), idx_next.max())) + 1, np.int64)
    pos_b[idx_b] = np.arange(idx_b.size)
    send_local, send_counts, recv_ids, recv_counts = [], [], [], []
    for s in range(world):
        a, b = ranges[s][0] * group_size, ranges[s][1] * group_size
        need = idx_next[a:b]                       # peer s's block-(b+1) rows, in its order
        src = pos_b[need] // chunk                 # their owners in block b
        sel = src == rank
        send_local.append(pos_b[need[sel]] - rank * chunk)
        send_counts.append(int(sel.sum()))
        if s == rank:
            for r in range(world):
                m = src == r
                recv_ids.append(need[m])
                recv_counts.append(int(m.sum()))
    return (np.concatenate(send_local), send_counts, np.concatenate(recv_ids), recv_counts)


def split_forward_a2a(runner, n_blocks: int, group_size: int, world: int, rank: int,
                      all_gather: Callable, all_to_all: Callable, alloc: Callable):
    """`split_forward` with an all-to-all of only the rows each rank needs next (about
    K/P rows in and out per rank and block instead of the all-gather's K): the ranks
    derive the per-peer row lists from the replicated schedule (runner.plan(b): block b's
    window-sort order).  The final block still all-gathers (the output is replicated).
    all_to_all(dst, src, dst_counts, src_counts): rows, rank-ordered chunks (NCCL / gloo
    all_to_all_single).  runner additionally: pack(y_local, local_idx) -> rows,
    unpack(rows, pillar_ids, dst) (dst[pillar_ids] = rows), alloc_rows(n)."""
    K = runner.begin()
    n_groups = K // group_size
    ranges, per = partition_groups(n_groups, world)
    g0, g1 = ranges[rank]
    y_local = alloc(per * group_size)
    y_all = alloc(world * per * group_size)
    if hasattr(runner, "exchange_tables_all"):
        tables = runner.exchange_tables_all(n_blocks, ranges, per, group_size, rank, world)
    else:
        tables = [runner.exchange_tables(b, ranges, per, group_size, rank, world) for b in range(n_blocks - 1)]
    x = runner.input()
    for b in range(n_blocks):
        runner.block(b, g0, g1, x, y_local)
        if b == n_blocks - 1:
            all_gather(y_all, y_local)
            runner.scatter(b, y_all, runner.out_buffer())
            break
        send_local, send_counts, recv_ids, recv_counts = tables[b]
        send = runner.pack(y_local, send_local)
        recv = runner.alloc_rows(int(sum(recv_counts)))
        all_to_all(recv, send, recv_counts, send_counts)
        x = runner.x_buffer()
        runner.unpack(recv, recv_ids, x)
    return runner.out_buffer()


def p2p_dest_rows(idx_b, idx_next, out_pos, ranges, per, group_size, rank, last):
    """The rank-tagged scatter rows of `split_forward_p2p` (what fwa_b200_split_p2p_setup
    builds on the device): row r of this rank's block-b range -> (rank owning its pillar in
    block b+1) << 28 | pillar id, or, for the last block, rank 0's output row."""
    import numpy as np
    a, e = ranges[rank][0] * group_size, ranges[rank][1] * group_size
    if last:
        return np.asarray(out_pos, np.int64)[a:e]
    idx_b = np.asarray(idx_b, np.int64)
    idx_next = np.asarray(idx_next, np.int64)
    pos = np.empty(int(max(idx_b.max(), idx_next.max())) + 1, np.int64)
    pos[idx_next] = np.arange(idx_next.size)
    pid = idx_b[a:e]
    return ((pos[pid] // (per * group_size)) << 28) | pid


def split_forward_p2p(runner, n_blocks: int, group_size: int, world: int, rank: int, barrier: Callable,
                      agree: Optional[Callable] = None):
    """runner: begin() -> K; p2p_setup(world, rank) (peer pointers + tables); input();
    x_buffer(); block_p2p(b, x); out_buffer().  barrier(): orders every rank's block b before
    any rank's block b+1 (stream-ordered).  agree: see DeviceRunner.p2p_setup.  Returns the
    output buffer (complete on rank 0)."""
    runner.begin()
    runner.p2p_setup(world, rank, agree) if agree is not None else runner.p2p_setup(world, rank)
    x = runner.input()
    for b in range(n_blocks):
        runner.block_p2p(b, x)
        barrier()
        x = runner.x_buffer()
    return runner.out_buffer()


def split_forward_p2p_emulated(runners, n_blocks: int):
    """`world` = len(runners) ranks of split_forward_p2p in ONE process (one GPU): every
    rank's runner has its own context, x buffer and output; the peers are plain local
    pointers and the ranks' blocks run in turn on one stream (that order is the barrier).
    Rank 0's output is returned."""
    world = len(runners)
    for r in runners:
        r.begin()
    xs = [r.x_buffer().data_ptr() for r in runners]
    outs = [r.out_buffer().data_ptr() for r in runners]
    for rk, r in enumerate(runners):
        r.ctx.split_p2p_setup(world, rk, xs, outs)
    for b in range(n_blocks):
        for r in runners:
            r.block_p2p(b, r.input() if b == 0 else r.x_buffer())
    return runners[0].out_buffer()


class DeviceRunner:
    """The C-ABI implementation (torch tensors for device memory)."""

    def __init__(self, ctx, d_coords, d_feats, cfg, same_stream=False, exchange_handles=None):
        """same_stream: the context runs on torch's current stream (created with it), so
        library kernels, torch index ops and NCCL collectives are stream-ordered and no host
        synchronisation is needed.  exchange_handles: see p2p_setup (world > 1)."""
        import torch
        self.ctx, self.cfg = ctx, cfg
        self.d_coords, self.d_feats = d_coords, d_feats
        self.n = d_coords.shape[0]
        dev = d_feats.device
        self.same_stream = same_stream
        self.exchange_handles = exchange_handles
        self._opened = []
        self._x_raw = self._out_raw = None
        if exchange_handles is not None:  # cudaMalloc'd (IPC-shareable) x buffer
            self._x_raw = ctx.alloc(self.n * cfg.d_model * 4)
            self.x = _device_view(self._x_raw, (self.n, cfg.d_model), dev)
        else:
            self.x = torch.empty((self.n, cfg.d_model), dtype=torch.float32, device=dev)
        self.out = None
        self.dev = dev

    def begin(self):
        import torch
        K = self.ctx.split_begin(self.d_coords.data_ptr(), self.n, self.cfg)
        if self.exchange_handles is not None:
            if self._out_raw is None:
                self._out_raw = self.ctx.alloc(K * self.cfg.d_model * 4)
            self.out = _device_view(self._out_raw, (K, self.cfg.d_model), self.dev)
        else:
            self.out = torch.empty((K, self.cfg.d_model), dtype=torch.float32, device=self.dev)
        return K

    def close(self):
        for p in self._opened:
            self.ctx.ipc_close(p)
        self._opened = []
        for p in (self._x_raw, self._out_raw):
            if p:
                self.ctx.free(p)
        self._x_raw = self._out_raw = None

    def input(self):
        return self.d_feats

    def x_buffer(self):
        return self.x

    def out_buffer(self):
        return self.out

    def block(self, b, g0, g1, x, y_local):
        self.ctx.split_block(b, g0, g1, x.data_ptr(), y_local.data_ptr())
        if not self.same_stream:
            self.ctx.sync_check()  # the library's stream -> torch's (collectives, index ops)

    # ---- peer-memory exchange (split_forward_p2p)
    def p2p_setup(self, world, rank, agree=None):
        """Peer pointers: this rank's own buffers alone, or -- with `exchange_handles`
        (rank-ordered all-gather of bytes objects, e.g. dist.all_gather_object) -- CUDA IPC
        mappings of every rank's cudaMalloc'd x and output buffers.  The mappings are made
        once per runner (the buffers do not move).  agree(ok) -> bool: every rank's verdict
        on its mappings (e.g. an all-reduce MIN), so a failure raises on ALL ranks alike
        instead of leaving the others waiting in the first inter-block barrier."""
        key = (world, rank, self.x.data_ptr(), self.out.data_ptr())
        if getattr(self, "_p2p_key", None) == key:
            self.ctx.split_p2p_setup(world, rank, self._p2p_xs, self._p2p_outs)
            return
        if world == 1:
            xs, outs = [self.x.data_ptr()], [self.out.data_ptr()]
        else:
            if self.exchange_handles is None:
                raise RuntimeError("split_forward_p2p with world > 1 needs exchange_handles")
            mine = (self.ctx.ipc_handle(self._x_raw), self.ctx.ipc_handle(self._out_raw))
            allh = self.exchange_handles(mine)
            xs, outs = [], []
            ok = True
            try:
                for r, (hx, ho) in enumerate(allh):
                    if r == rank:
                        xs.append(self._x_raw)
                        outs.append(self._out_raw)
                    else:
                        xs.append(self.ctx.ipc_open(hx))
                        self._opened.append(xs[-1])
                        outs.append(self.ctx.ipc_open(ho))
                        self._opened.append(outs[-1])
            except Exception:  # noqa: BLE001 -- reported through `agree`
                ok = False
            if agree is not None:
                ok = agree(ok)
            if not ok:
                raise RuntimeError("peer-memory split: CUDA IPC mapping failed on at least one rank")
        self.ctx.split_p2p_setup(world, rank, xs, outs)
        self._p2p_key, self._p2p_xs, self._p2p_outs = key, xs, outs

    def block_p2p(self, b, x):
        self.ctx.split_block_p2p(b, x.data_ptr() if hasattr(x, "data_ptr") else int(x))

    def scatter(self, b, y_all, dst):
        self.ctx.split_scatter(b, y_all.data_ptr(), dst.data_ptr())

    # ---- all-to-all exchange (split_forward_a2a)
    def exchange_tables_all(self, n_blocks, ranges, per, group_size, rank, world):
        """exchange_tables() of every block transition on the device (torch ops over the
        schedule's window-sort orders, once per scene); the per-peer counts (the
        collective's splits) come back to the host in ONE copy."""
        import torch
        K = self.out.shape[0]
        plans = []
        for i in range(n_blocks):
            p32 = torch.empty(K, dtype=torch.int32, device=self.dev)
            self.ctx.split_plan_device(i, p32.data_ptr())
            plans.append(p32)
        self.ctx.sync_check()
        plans = [p.long() for p in plans]
        chunk = per * group_size
        a, e = ranges[rank][0] * group_size, ranges[rank][1] * group_size
        pos_b = torch.empty(int(self.n), dtype=torch.long, device=self.dev)
        ar = torch.arange(K, device=self.dev)
        out, counts = [], []
        for b in range(n_blocks - 1):
            idx_b, idx_n = plans[b], plans[b + 1]
            pos_b[idx_b] = ar
            pos_n = pos_b[idx_n]                      # block-b position of block-(b+1) row k
            src = torch.div(pos_n, chunk, rounding_mode="floor")
            send_k = torch.nonzero(src == rank).squeeze(1)  # ascending k = grouped by destination
            send_local = pos_n[send_k] - rank * chunk
            my_src = src[a:e]
            recv_ids = idx_n[a:e][torch.argsort(my_src, stable=True)]
            counts.append(torch.bincount(torch.div(send_k, chunk, rounding_mode="floor"), minlength=world))
            counts.append(torch.bincount(my_src, minlength=world))
            out.append((send_local, recv_ids))
        c = torch.stack(counts).cpu().tolist() if counts else []
        return [(sl, c[2 * i], ri, c[2 * i + 1]) for i, (sl, ri) in enumerate(out)]

    def pack(self, y_local, local_idx):
        return y_local.index_select(0, local_idx)

    def unpack(self, rows, pillar_ids, dst):
        import torch
        dst.index_copy_(0, pillar_ids, rows)
        if not self.same_stream:
            torch.cuda.synchronize(self.dev)  # before the next block kernel (library stream) reads dst

    def alloc_rows(self, n):
        import torch
        return torch.empty((n, self.cfg.d_model), dtype=torch.float32, device=self.dev)


def _device_view(ptr, shape, dev):
    """A torch float32 tensor over raw device memory (no ownership)."""
    import torch

    class _Arr:
        __cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f4", "data": (int(ptr), False),
                                    "version": 3, "strides": None}
    return torch.as_tensor(_Arr(), device=dev)
