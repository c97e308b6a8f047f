"""Cross-GPU decode host logic on CPU: placement, locality-first
survivor choice, pointer tables, the handle exchange, and the staged (NCCL-style) baseline's
exchange lists, over gloo at world size 2.  Expected bytes come from the oracle only: a
pointer table is "resolved" back to (rank, slot) and the oracle decodes what it points at.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import matrices as mx
from oracle import rs
from paper_2108_02692_b200.peer import Placement, Plan, PeerDecoder, exchange_lists, staged_gather

FAKE = 1 << 40          # fake per-rank base addresses: rank r's storage at r * FAKE


def codewords(seed, S, n, p, B, g):
    out = []
    for s in range(S):
        d = synth.stripe_data(seed, s, n, B)
        out.append(np.concatenate([d, rs.encode(g, n, d)]))
    return np.stack(out)                                  # [S][n+p][B]


def storage_of(pl, rank, cw):
    S, _, B = cw.shape
    st = np.zeros((S, pl.slots, B), dtype=np.uint8)
    for s in range(S):
        for j in pl.blocks_of(rank, s):
            st[s, pl.slot(s, j)] = cw[s, j]
    return st


def erasures_fn(seed, n, p, e):
    return lambda s: synth.erasure_pattern(seed, s, n + p, e)


def test_placement_is_a_bijection():
    for n, p, world in [(10, 4, 1), (10, 4, 2), (10, 4, 8), (20, 4, 3), (4, 2, 8)]:
        pl = Placement(n, p, world, 17)
        for s in range(17):
            seen = set()
            for j in range(n + p):
                o, k = pl.owner(s, j), pl.slot(s, j)
                assert 0 <= o < world and 0 <= k < pl.slots
                assert (o, k) not in seen
                seen.add((o, k))
                assert pl.blocks_of(o, s)[k] == j
        homes = sorted(s for r in range(world) for s in pl.home_stripes(r))
        assert homes == list(range(17))


def test_survivors_prefer_local_blocks():
    n, p, world = 10, 4, 4
    pl = Placement(n, p, world, 8)
    for s in range(8):
        h = pl.home(s)
        for erased in ([], [0], [1, 2], [3, 5, 7]):
            sv = pl.choose_survivors(s, erased)
            assert len(sv) == n and sv == sorted(sv) and not set(sv) & set(erased)
            alive = [j for j in range(n + p) if j not in erased]
            local_alive = [j for j in alive if pl.owner(s, j) == h]
            assert sum(pl.owner(s, j) == h for j in sv) == min(n, len(local_alive))
        with pytest.raises(ValueError):
            pl.choose_survivors(s, [0, 1, 2, 3, 4])


@pytest.mark.parametrize("world,e", [(1, 4), (2, 4), (3, 2), (8, 4)])
def test_tables_resolve_to_the_oracle_decode(world, e):
    # every rank's table, resolved through the fake bases, reads survivors whose oracle
    # decode equals the erased blocks of the codeword
    n, p, B, S = 10, 4, 64, 12
    g = mx.coding_matrix(n, p)
    cw = codewords(31, S, n, p, B, g)
    pl = Placement(n, p, world, S)
    stores = [storage_of(pl, r, cw) for r in range(world)]
    er = erasures_fn(31, n, p, e)
    bases = [r * FAKE for r in range(world)]
    for r in range(world):
        plan = Plan(pl, r, er)
        assert plan.stripes == pl.home_stripes(r) and plan.e == e
        tin = plan.in_table(bases, B)
        tout = plan.out_table(7 * FAKE, B)
        assert (tout.reshape(-1) == 7 * FAKE + np.arange(len(plan.stripes) * e) * B).all()
        for i, s in enumerate(plan.stripes):
            erased, surv = plan.keys[plan.key_of[i]]
            assert list(erased) == synth.erasure_pattern(31, s, n + p, e)
            blocks = []
            for c in range(n):
                rank, off = divmod(int(tin[i, c]), FAKE)
                row, rem = divmod(off, pl.slots * B)
                slot, z = divmod(rem, B)
                assert row == s and z == 0
                blocks.append(stores[rank][row, slot])
            rows = mx.decode_rows_from(g, n, list(erased), list(surv))
            assert (rs.decode(rows, np.stack(blocks)) == cw[s, list(erased)]).all()
        rem, tot = plan.remote_reads()
        assert tot == n * len(plan.stripes) and (rem == 0) == (world == 1)


def test_groups_partition_the_stripes():
    pl = Placement(10, 4, 2, 40)
    plan = Plan(pl, 1, erasures_fn(3, 10, 4, 4))
    ids, off = plan.groups()
    assert off[0] == 0 and off[-1] == len(plan.stripes) and sorted(ids.tolist()) == list(range(20))
    for k in range(len(plan.keys)):
        assert all(plan.key_of[i] == k for i in ids[off[k]:off[k + 1]])


def test_exchange_lists_match_between_ranks():
    n, p, world, S = 10, 4, 4, 24
    pl = Placement(n, p, world, S)
    er = erasures_fn(8, n, p, 3)
    lists = [exchange_lists(pl, r, er) for r in range(world)]
    for a in range(world):
        for b in range(world):
            if a != b:
                assert lists[a][0][b] == lists[b][1][a]      # a sends to b what b receives
    for r in range(world):                                 # every remote survivor arrives once
        plan = Plan(pl, r, er)
        want = sorted((s, j) for i, s in enumerate(plan.stripes)
                      for j in plan.keys[plan.key_of[i]][1] if pl.owner(s, j) != r)
        got = sorted(x for q in lists[r][1].values() for x in q)
        assert got == want


# ---- world size 2 over gloo ----------------------------------------------------------------

class FakeX:
    """Stands in for the C ABI's peer calls: the handle carries the exporter's rank and the
    "mapped" address is that rank's fake base."""

    def __init__(self, rank):
        self.rank, self.closed = rank, []

    def xslp_peer_export(self, t):
        return b"rank%03d" % self.rank + bytes(121)

    def xslp_peer_open(self, h):
        return int(h[4:7]) * FAKE

    def xslp_peer_close(self, a):
        self.closed.append(a)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, p, B, S = 10, 4, 64, 10
        g = mx.coding_matrix(n, p)
        cw = codewords(41, S, n, p, B, g)          # every rank can regenerate every codeword
        pl = Placement(n, p, world, S)
        er = erasures_fn(41, n, p, 3)
        plan = Plan(pl, rank, er)
        storage = torch.from_numpy(storage_of(pl, rank, cw))
        # staged baseline: remote survivors arrive by point-to-point messages
        staging = torch.zeros((len(plan.stripes), n, B), dtype=torch.uint8)
        staged_gather(pl, plan, storage, staging, er, dist)
        ok_staged = True
        for i, s in enumerate(plan.stripes):
            erased, surv = plan.keys[plan.key_of[i]]
            rows = mx.decode_rows_from(g, n, list(erased), list(surv))
            ok_staged &= bool((rs.decode(rows, staging[i].numpy()) == cw[s, list(erased)]).all())
        # peer path: handles exchanged with all_gather_object, tables over the mapped bases
        out = torch.zeros((len(plan.stripes), plan.e, B), dtype=torch.uint8)
        fx = FakeX(rank)
        dec = PeerDecoder(fx, pl, storage, out, plan, progs=[None] * len(plan.keys), dist=dist)
        bases = dec.bases
        ok_bases = bases[rank] == storage.data_ptr() and all(
            bases[r] == r * FAKE for r in range(world) if r != rank)
        tin = dec.in_tbl.view(len(plan.stripes), n).numpy()
        ok_peer = True
        for i, s in enumerate(plan.stripes):
            for c, j in enumerate(plan.keys[plan.key_of[i]][1]):
                o = pl.owner(s, j)
                want = bases[o] + (s * pl.slots + pl.slot(s, j)) * B
                ok_peer &= int(tin[i, c]) == want
        dec.close()
        ok_close = sorted(fx.closed) == sorted(r * FAKE for r in range(world) if r != rank)
        q.put((rank, ok_staged, ok_bases, ok_peer, ok_close))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_staged_and_peer_tables():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=180) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert res == [(0, True, True, True, True), (1, True, True, True, True)]
