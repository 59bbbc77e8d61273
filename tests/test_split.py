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
from paper_2301_08739_b200.split import partition_groups, split_forward

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


def test_partition_groups():
    r, per = partition_groups(10, 3)
    assert r == [(0, 4), (4, 8), (8, 10)] and per == 4
    r, per = partition_groups(2, 4)
    assert r == [(0, 1), (1, 2), (2, 2), (2, 2)] and per == 1


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
