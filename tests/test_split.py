"""Config 4 host logic: one scene split by group ranges across ranks with an all-gather
between blocks (paper_2301_08739_b200/split.py).

CPU: world_size 2 over gloo with an oracle runner (the C restatement computes each rank's
groups) -- must equal the single-process oracle backbone bit for bit.
GPU: the C-ABI runner, single process emulating 1 and 3 ranks -- bitwise equal to
run_backbone (rows are independent of their tile position)."""
import os

import numpy as np
import pytest

import oracle as O
import paper_2301_08739_b200 as F
from paper_2301_08739_b200.split import (exchange_tables, p2p_dest_rows, partition_groups, split_forward,
                                         split_forward_a2a, split_forward_p2p)

D, H, DFF, G, NB = 16, 4, 32, 16, 4


def _scene(seed=11, n=1000):
    rng = np.random.default_rng(seed)
    c = np.round(rng.uniform(-20, 20, size=(n, 2)) / 0.32) * 0.32 + 0.16
    c = np.unique(c, axis=0)
    f = rng.normal(size=(c.shape[0], D)).astype(np.float32)
    return c, f


class OracleRunner:
    """CPU runner: schedule from the NumPy window-sort oracle, blocks from the C restatement."""

    def __init__(self, coords, feats, blob):
        self.c, self.f, self.blob = coords, feats, blob
        self.rec = len(blob) // NB

    def begin(self):
        n = self.c.shape[0]
        w = 9 * 0.32
        p0 = O.np_sort(self.c, w, w, 0, 0)
        nk = (n // G) * G
        kept = np.zeros(n, bool)
        kept[p0[:nk]] = True
        self.idx = []
        for b in range(NB):
            ay, sh = (b % 4) >= 2, b % 2
            full = O.np_sort(self.c, w, w, sh, ay)
            self.idx.append(full[kept[full]])
        rank = np.cumsum(kept) - 1
        self.out_pos = rank[self.idx[NB - 1]]
        self.pe = O.port_positional_embedding(self.c, D)
        self.x = np.zeros_like(self.f)
        self.out = np.zeros((nk, D), np.float32)
        return nk

    def input(self):
        return self.f

    def x_buffer(self):
        return self.x

    def out_buffer(self):
        return self.out

    def block(self, b, g0, g1, x, y_local):
        rows = self.idx[b][g0 * G:g1 * G]
        if len(rows):
            rec = self.blob[b * self.rec:(b + 1) * self.rec]
            y_local[:len(rows)] = O.port_block_forward(x[rows], self.pe[rows], g1 - g0, rec)

    def scatter(self, b, y_all, dst):
        pos = self.out_pos if b == NB - 1 else self.idx[b]
        dst[pos] = y_all[:len(pos)]

    # all-to-all exchange (split_forward_a2a)
    def exchange_tables(self, b, ranges, per, group_size, rank, world):
        return exchange_tables(self.idx[b], self.idx[b + 1], ranges, per, group_size, rank, world)

    def pack(self, y_local, local_idx):
        return y_local[local_idx]

    def unpack(self, rows, pillar_ids, dst):
        dst[pillar_ids] = rows

    def alloc_rows(self, n):
        return np.zeros((n, D), np.float32)


def test_partition_groups():
    r, per = partition_groups(10, 3)
    assert r == [(0, 4), (4, 8), (8, 10)] and per == 4
    r, per = partition_groups(2, 4)
    assert r == [(0, 1), (1, 2), (2, 2), (2, 2)] and per == 1


def _gloo_worker_a2a(rank, world, port, coords, feats, blob, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def all_gather(dst, src):
            parts = [torch.empty_like(torch.from_numpy(src)) for _ in range(world)]
            dist.all_gather(parts, torch.from_numpy(src))
            dst[:] = torch.cat(parts).numpy()

        def all_to_all(dst, src, dst_counts, src_counts):
            out = torch.from_numpy(dst)
            dist.all_to_all_single(out, torch.from_numpy(np.ascontiguousarray(src)), dst_counts, src_counts)

        runner = OracleRunner(coords, feats, blob)
        out = split_forward_a2a(runner, NB, G, world, rank, all_gather, all_to_all,
                                lambda rows: np.zeros((rows, D), np.float32))
        q.put((rank, out.copy()))
    finally:
        dist.destroy_process_group()


def _gloo_worker(rank, world, port, coords, feats, blob, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def all_gather(dst, src):
            parts = [torch.empty_like(torch.from_numpy(src)) for _ in range(world)]
            dist.all_gather(parts, torch.from_numpy(src))
            dst[:] = torch.cat(parts).numpy()

        runner = OracleRunner(coords, feats, blob)
        out = split_forward(runner, NB, G, world, rank, all_gather,
                            lambda rows: np.zeros((rows, D), np.float32))
        q.put((rank, out.copy()))
    finally:
        dist.destroy_process_group()


def test_split_gloo_world2_equals_single_process():
    import torch.multiprocessing as mp
    coords, feats = _scene()
    cfg = O.make_cfg(d_model=D, n_heads=H, d_ff=DFF, group_size=G, n_blocks=NB)
    blob = F.init_backbone_params(F.FwaConfig(d_model=D, n_heads=H, d_ff=DFF, group_size=G, n_blocks=NB), 5)
    want = O.port_run_backbone(coords, feats, cfg, blob)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, coords, feats, blob, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    for r in range(2):
        assert np.array_equal(outs[r], want["features"]), r


def test_exchange_tables_cover_every_next_block_row():
    """Every rank receives exactly its next-block rows, each from its block-b owner."""
    rng = np.random.default_rng(3)
    K, world = 37 * G, 3
    kept = rng.permutation(K + 5)[:K]  # both blocks order the same kept pillars
    idx_b, idx_n = rng.permutation(kept), rng.permutation(kept)
    ranges, per = partition_groups(K // G, world)
    tabs = [exchange_tables(idx_b, idx_n, ranges, per, G, r, world) for r in range(world)]
    for s_ in range(world):
        a, b = ranges[s_][0] * G, ranges[s_][1] * G
        got = np.concatenate([tabs[s_][2]])
        assert sorted(got.tolist()) == sorted(idx_n[a:b].tolist())
        # what s_ receives from r is what r sends to s_, in the same order
        off = np.cumsum([0] + tabs[s_][3])
        for r in range(world):
            s_off = np.cumsum([0] + tabs[r][1])
            sent_local = tabs[r][0][s_off[s_]:s_off[s_ + 1]]
            sent_ids = idx_b[sent_local + r * per * G]
            assert np.array_equal(sent_ids, got[off[r]:off[r + 1]])


@pytest.mark.parametrize("world", [2, 3])
def test_split_a2a_gloo_equals_single_process(world):
    """The all-to-all exchange (only the rows each rank needs next) == the single-process
    oracle backbone, bit for bit, at world sizes 2 and 3 over gloo."""
    import torch.multiprocessing as mp
    coords, feats = _scene()
    cfg = O.make_cfg(d_model=D, n_heads=H, d_ff=DFF, group_size=G, n_blocks=NB)
    blob = F.init_backbone_params(F.FwaConfig(d_model=D, n_heads=H, d_ff=DFF, group_size=G, n_blocks=NB), 5)
    want = O.port_run_backbone(coords, feats, cfg, blob)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + (os.getpid() % 1000) + world
    procs = [ctx.Process(target=_gloo_worker_a2a, args=(r, world, port, coords, feats, blob, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    for r in range(world):
        assert np.array_equal(outs[r], want["features"]), r


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 3])
def test_split_device_runner_equals_run_backbone(world):
    import torch
    from paper_2301_08739_b200.split import DeviceRunner
    ps = F.make_pillars(F.SCENES["F10"], 42)
    cfg = F.FwaConfig()
    ctx = F.Context(0, precision="bf16")
    ctx.load_params(cfg, F.init_backbone_params(cfg, 42))
    want = ctx.run_backbone(F.PillarSet(ps.coords, ps.features.astype(np.float32)), cfg)
    dev = torch.device("cuda", 0)
    dc = torch.from_numpy(ps.coords).to(dev)
    df = torch.from_numpy(ps.features.astype(np.float32)).to(dev)
    runner = DeviceRunner(ctx, dc, df, cfg)
    # emulate `world` ranks in one process: every "rank" computes its range into its own
    # slice of the gathered buffer (the all-gather's rank-ordered concatenation)
    K = runner.begin()
    n_groups = K // cfg.group_size
    ranges, per = partition_groups(n_groups, world)
    y_all = torch.zeros((world * per * cfg.group_size, 128), dtype=torch.float32, device=dev)
    x = runner.input()
    for b in range(cfg.n_blocks):
        for r in range(world):
            g0, g1 = ranges[r]
            y_loc = y_all[r * per * cfg.group_size:(r + 1) * per * cfg.group_size]
            runner.block(b, g0, g1, x, y_loc)
        dst = runner.out_buffer() if b == cfg.n_blocks - 1 else runner.x_buffer()
        runner.scatter(b, y_all, dst)
        x = dst
    out = runner.out_buffer()
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), want.features)


@pytest.mark.gpu
def test_split_a2a_device_runner_equals_run_backbone():
    """The all-to-all exchange with the C-ABI runner (plan / pack / unpack on the device),
    one rank: bitwise equal to run_backbone."""
    import torch
    from paper_2301_08739_b200.split import DeviceRunner
    ps = F.make_pillars(F.SCENES["F10"], 42)
    cfg = F.FwaConfig()
    ctx = F.Context(0, precision="bf16")
    ctx.load_params(cfg, F.init_backbone_params(cfg, 42))
    want = ctx.run_backbone(F.PillarSet(ps.coords, ps.features.astype(np.float32)), cfg)
    dev = torch.device("cuda", 0)
    runner = DeviceRunner(ctx, torch.from_numpy(ps.coords).to(dev),
                          torch.from_numpy(ps.features.astype(np.float32)).to(dev), cfg)
    out = split_forward_a2a(runner, cfg.n_blocks, cfg.group_size, 1, 0,
                            lambda dst, src: dst.copy_(src),
                            lambda dst, src, dc, sc: dst.copy_(src),
                            lambda rows: torch.zeros((rows, 128), dtype=torch.float32, device=dev))
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), want.features)


# ----------------------------------------------------------------------------- peer memory

class SharedPeerOracleRunner(OracleRunner):
    """split_forward_p2p on CPU: every rank's x buffer and output live in shared memory (the
    stand-in for NVLink peer memory); block_p2p computes the rank's range with the C
    restatement and writes each output row into the buffer of the rank that consumes it
    next, per p2p_dest_rows -- exactly the rank-tagged rows the device tables hold."""

    def __init__(self, coords, feats, blob, shm_x, shm_out):
        super().__init__(coords, feats, blob)
        self.shm_x, self.shm_out = shm_x, shm_out

    def begin(self):
        nk = super().begin()
        self.peers_x = [np.frombuffer(b, np.float32).reshape(-1, D) for b in self.shm_x]
        self.peers_out = [np.frombuffer(b, np.float32).reshape(-1, D) for b in self.shm_out]
        return nk

    def p2p_setup(self, world, rank):
        self.world, self.rank = world, rank
        n_groups = self.out.shape[0] // G
        self.ranges, self.per = partition_groups(n_groups, world)

    def x_buffer(self):
        return self.peers_x[self.rank]

    def out_buffer(self):
        return self.peers_out[self.rank]

    def block_p2p(self, b, x):
        g0, g1 = self.ranges[self.rank]
        rows = self.idx[b][g0 * G:g1 * G]
        if not len(rows):
            return
        rec = self.blob[b * self.rec:(b + 1) * self.rec]
        y = O.port_block_forward(x[rows], self.pe[rows], g1 - g0, rec)
        last = b == NB - 1
        tags = p2p_dest_rows(self.idx[b], None if last else self.idx[b + 1], self.out_pos, self.ranges,
                             self.per, G, self.rank, last)
        if last:
            self.peers_out[0][tags] = y
            return
        for k, t in enumerate(tags):
            self.peers_x[int(t) >> 28][int(t) & 0x0FFFFFFF] = y[k]


def _gloo_worker_p2p(rank, world, port, coords, feats, blob, shm_x, shm_out, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        runner = SharedPeerOracleRunner(coords, feats, blob, shm_x, shm_out)
        out = split_forward_p2p(runner, NB, G, world, rank, dist.barrier)
        q.put((rank, out.copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_split_p2p_gloo_equals_single_process(world):
    """The peer-memory exchange (each block's rows written straight into the consumer
    rank's buffer, a barrier between blocks): rank 0's output == the single-process oracle
    backbone, bit for bit, at world sizes 2 and 3 (gloo barrier, shared-memory peers)."""
    import torch.multiprocessing as mp
    coords, feats = _scene()
    cfg = O.make_cfg(d_model=D, n_heads=H, d_ff=DFF, group_size=G, n_blocks=NB)
    blob = F.init_backbone_params(F.FwaConfig(d_model=D, n_heads=H, d_ff=DFF, group_size=G, n_blocks=NB), 5)
    want = O.port_run_backbone(coords, feats, cfg, blob)
    ctx = mp.get_context("spawn")
    n, nk = coords.shape[0], want["features"].shape[0]
    shm_x = [ctx.RawArray("f", n * D) for _ in range(world)]
    shm_out = [ctx.RawArray("f", nk * D) for _ in range(world)]
    q = ctx.Queue()
    port = 31500 + (os.getpid() % 1000) + world
    procs = [ctx.Process(target=_gloo_worker_p2p, args=(r, world, port, coords, feats, blob, shm_x, shm_out, q))
             for r in range(world)]
    for p in procs:
        p.start()
    outs = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    assert np.array_equal(outs[0], want["features"])


def test_p2p_dest_rows_partition_every_next_block_row():
    """Every pillar of a rank's block-b range is tagged with the rank that holds it in block
    b+1: over all ranks the tags route each next-block row to exactly its owner."""
    rng = np.random.default_rng(8)
    K, world = 41 * G, 3
    kept = rng.permutation(K + 7)[:K]
    idx_b, idx_n = rng.permutation(kept), rng.permutation(kept)
    ranges, per = partition_groups(K // G, world)
    got = {}
    for r in range(world):
        for t in p2p_dest_rows(idx_b, idx_n, None, ranges, per, G, r, False):
            got[int(t) & 0x0FFFFFFF] = int(t) >> 28
    assert len(got) == K
    for s_ in range(world):
        a, b = ranges[s_][0] * G, ranges[s_][1] * G
        assert all(got[int(p)] == s_ for p in idx_n[a:b])


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 3])
def test_split_p2p_device_emulated_equals_run_backbone(world):
    """The C-ABI peer-memory split, `world` ranks emulated in one process on one GPU (each
    rank its own context, x buffer and output; peers = local pointers): rank 0's output is
    bitwise equal to run_backbone (rows are independent of their tile position)."""
    import torch
    from paper_2301_08739_b200.split import DeviceRunner, split_forward_p2p_emulated
    ps = F.make_pillars(F.SCENES["F10"], 42)
    cfg = F.FwaConfig()
    blob = F.init_backbone_params(cfg, 42)
    ref_ctx = F.Context(0, precision="bf16")
    ref_ctx.load_params(cfg, blob)
    want = ref_ctx.run_backbone(F.PillarSet(ps.coords, ps.features.astype(np.float32)), cfg)
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(dev)
    with torch.cuda.stream(st):
        dc = torch.from_numpy(ps.coords).to(dev)
        df = torch.from_numpy(ps.features.astype(np.float32)).to(dev)
        runners = []
        for _ in range(world):
            c = F.Context(0, stream=st.cuda_stream, precision="bf16")
            c.load_params(cfg, blob)
            runners.append(DeviceRunner(c, dc, df, cfg, same_stream=True))
        out = split_forward_p2p_emulated(runners, cfg.n_blocks)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), want.features)
