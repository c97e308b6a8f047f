"""Cross-GPU decode: survivor blocks resident on other GPUs of the box.

A stripe's n+p blocks are spread over the ranks (one process per GPU).  Rank h(s) decodes
stripe s.  Its survivors are read IN PLACE: every rank exports its block storage
(xslp_peer_export), every rank maps the others' (xslp_peer_open, NVLink P2P), and the
decode kernel's input pointer table names local or peer addresses per block.  The
straight-line kernel's strip loads then pull remote strips over NVLink 5
/ NVSwitch and feed the XOR network directly (H9): the exchange is fused into the decode,
overlapping transfer and XORs tile by tile, with no staging buffer written and re-read.

`staged_gather` is the baseline it replaces: move the remote survivors into a local staging
buffer with NCCL point-to-point (torch.distributed batch_isend_irecv), then decode locally.

Placement (rotating, as erasure-coded stores spread a stripe over failure domains): block j
of global stripe s lives on rank (s + j) % world, in slot j // world of row s of that rank's
storage tensor [S][slots][B], slots = ceil((n+p)/world).  Stripe s is decoded by rank
s % world into row s // world of its output [S_home][e][B].  When fewer than p blocks are
erased the decode may read any n survivors (MDS); `choose_survivors` takes the
decoding rank's own blocks first, so fewer bytes cross NVLink.

The host logic here (placement, survivor choice, pattern grouping, pointer tables, staged
exchange lists) is plain Python + numpy and is tested on CPU with gloo at world size 2
(tests/test_peer.py); device work goes through the C ABI only.
"""
import numpy as np


class Placement:
    def __init__(self, n, p, world, stripes):
        if world < 1 or n < 1 or p < 0 or stripes < 0:
            raise ValueError("bad placement arguments")
        self.n, self.p, self.world, self.stripes = n, p, world, stripes
        self.slots = -(-(n + p) // world)

    def owner(self, s, j):
        return (s + j) % self.world

    def slot(self, s, j):
        return j // self.world

    def blocks_of(self, rank, s):
        """Block indices of stripe s stored on `rank` (ascending; slot k holds the k-th)."""
        return [j for j in range(self.n + self.p) if self.owner(s, j) == rank]

    def home(self, s):
        return s % self.world

    def home_stripes(self, rank):
        return list(range(rank, self.stripes, self.world))

    def home_index(self, s):
        return s // self.world

    def storage_shape(self, B):
        return (self.stripes, self.slots, B)

    def choose_survivors(self, s, erased):
        """n non-erased blocks of stripe s, the decoding rank's own first, ascending."""
        erased = set(erased)
        if len(erased) > self.p:
            raise ValueError("unrecoverable")
        h = self.home(s)
        alive = [j for j in range(self.n + self.p) if j not in erased]
        pick = sorted(alive, key=lambda j: (self.owner(s, j) != h, j))[:self.n]
        return sorted(pick)


class Plan:
    """What rank `rank` decodes: its home stripes, each stripe's (erased, survivors) key,
    the distinct keys (one compiled program each) and the per-stripe key index."""

    def __init__(self, placement, rank, erasures):
        """erasures: callable s -> erased block indices of global stripe s."""
        self.pl, self.rank = placement, rank
        self.stripes = placement.home_stripes(rank)
        self.keys, self.key_of = [], []
        index = {}
        for s in self.stripes:
            er = tuple(sorted(erasures(s)))
            sv = tuple(placement.choose_survivors(s, er))
            k = index.setdefault((er, sv), len(self.keys))
            if k == len(self.keys):
                self.keys.append((er, sv))
            self.key_of.append(k)
        ne = {len(k[0]) for k in self.keys}
        if len(ne) > 1:
            raise ValueError("all stripes of one decode must erase the same number of blocks")
        self.e = ne.pop() if ne else 0

    def remote_reads(self):
        """(remote survivor blocks, all survivor blocks) read by this rank's decode."""
        rem = tot = 0
        for s, k in zip(self.stripes, self.key_of):
            for j in self.keys[k][1]:
                tot += 1
                rem += self.pl.owner(s, j) != self.rank
        return rem, tot

    def in_table(self, bases, B):
        """int64 [S_home][n]: address of survivor block survivors[c] of each home stripe,
        bases[r] = address (local or mapped peer) of rank r's storage tensor."""
        pl = self.pl
        t = np.zeros((len(self.stripes), pl.n), dtype=np.int64)
        for i, (s, k) in enumerate(zip(self.stripes, self.key_of)):
            for c, j in enumerate(self.keys[k][1]):
                t[i, c] = bases[pl.owner(s, j)] + ((s * pl.slots + pl.slot(s, j)) * B)
        return t

    def out_table(self, out_base, B):
        """int64 [S_home][e]: row i of the [S_home][e][B] output at out_base."""
        S, e = len(self.stripes), self.e
        return (out_base + np.arange(S * e, dtype=np.int64) * B).reshape(S, e)

    def groups(self):
        """(stripe ids per key concatenated, offsets) for xslp_decode_batch_grouped."""
        key = np.asarray(self.key_of, dtype=np.int64)
        order = np.argsort(key, kind="stable").astype(np.int32)
        counts = np.bincount(key, minlength=len(self.keys)) if len(key) else np.zeros(len(self.keys), np.int64)
        off = np.zeros(len(self.keys) + 1, dtype=np.int32)
        off[1:] = np.cumsum(counts)
        return order, off


def exchange_lists(placement, rank, erasures):
    """Staged (baseline) exchange: for every other rank q, the (stripe, block) pairs this rank
    must SEND to q and RECEIVE from q, in one canonical order both sides derive alike."""
    pl = placement
    send = {q: [] for q in range(pl.world) if q != rank}
    recv = {q: [] for q in range(pl.world) if q != rank}
    for s in range(pl.stripes):
        h = pl.home(s)
        er = tuple(sorted(erasures(s)))
        for j in pl.choose_survivors(s, er):
            o = pl.owner(s, j)
            if o == h:
                continue
            if o == rank:
                send[h].append((s, j))
            elif h == rank:
                recv[o].append((s, j))
    return send, recv


class StagedGather:
    """Baseline: copy every survivor of a rank's home stripes into staging [S_home][n][B]
    (local ones by one device gather, remote ones by NCCL / gloo point-to-point), so a local
    decode can follow.  The index lists are built once; `run()` moves one step's bytes."""

    def __init__(self, placement, plan, storage, staging, erasures, X=None):
        """X: the binding; when given, local survivors are copied by an identity program
        (one 8-strip block in, the same block out) over block pointer tables -- one launch."""
        import numpy as np
        import torch
        pl, rank = placement, plan.rank
        self.pl, self.storage, self.staging, self.X = pl, storage, staging, X
        row = {s: i for i, s in enumerate(plan.stripes)}
        col = {}
        src, dst = [], []
        n = staging.shape[1]
        for i, (s, k) in enumerate(zip(plan.stripes, plan.key_of)):
            for c, j in enumerate(plan.keys[k][1]):
                col[(s, j)] = c
                if pl.owner(s, j) == rank:
                    src.append(s * pl.slots + pl.slot(s, j))
                    dst.append(i * n + c)
        self.src = torch.tensor(src, dtype=torch.long, device=storage.device)
        self.dst = torch.tensor(dst, dtype=torch.long, device=staging.device)
        if X is not None and src:
            B = staging.shape[-1]
            self.copy = X.xslp_compile(np.eye(8, dtype=np.uint8), kernel="straight", threads=128,
                                       block_bytes_hint=B)
            self.tin = self.src * B + storage.data_ptr()
            self.tout = self.dst * B + staging.data_ptr()
        send, recv = exchange_lists(pl, rank, erasures)
        self.sends = [(q, storage[s, pl.slot(s, j)]) for q, lst in send.items() for (s, j) in lst]
        self.recvs = [(q, staging[row[s], col[(s, j)]]) for q, lst in recv.items() for (s, j) in lst]

    def run(self, dist, group=None, stream=None):
        B = self.staging.shape[-1]
        if len(self.src) and self.X is not None:
            self.X.xslp_encode_batch(self.copy, self.tin, self.tout, len(self.src), B, stream=stream)
        elif len(self.src):
            self.staging.view(-1, B)[self.dst] = self.storage.view(-1, B)[self.src]
        ops = [dist.P2POp(dist.isend, t, q, group) for q, t in self.sends]
        ops += [dist.P2POp(dist.irecv, t, q, group) for q, t in self.recvs]
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()


def staged_gather(placement, plan, storage, staging, erasures, dist, group=None):
    """One-shot form of StagedGather."""
    StagedGather(placement, plan, storage, staging, erasures).run(dist, group)


class PeerDecoder:
    """Maps every rank's block storage on this rank's device and decodes this rank's home
    stripes straight from local + peer memory (one grouped launch, or a single batch launch
    when all home stripes share one program)."""

    def __init__(self, X, placement, storage, out, plan, progs, dist=None, group=None, multi=None,
                 tma=False):
        """multi: optional X.Multi over `progs` (fused multi-program kernels).  By default peer
        blocks are read by the LDG straight-line kernels (plain loads over P2P mappings, the
        path validated on real NVLink); tma=True (opt-in) lets TMA-staged kernels -- PIPE
        programs (compile_plan(..., kernel="pipe")) and the fused multi-program kernels --
        bulk-copy peer strips (cp.async.bulk from the mapped addresses)."""
        import torch
        self.X, self.pl, self.plan, self.progs = X, placement, plan, progs
        if multi is not None and placement.world > 1 and not tma:
            raise ValueError("the fused multi-program kernels read peer blocks only with tma=True")
        self.tma = tma
        self.multi = multi
        B = storage.shape[-1]
        self.B = B
        world = placement.world
        mine = X.xslp_peer_export(storage)
        if world > 1:
            handles = [None] * world
            dist.all_gather_object(handles, mine, group=group)
        else:
            handles = [mine]
        self.mapped = []
        bases = []
        for r, h in enumerate(handles):
            if r == plan.rank:
                bases.append(storage.data_ptr())
            else:
                a = X.xslp_peer_open(h)
                self.mapped.append(a)
                bases.append(a)
        self.bases = bases
        self.in_tbl = torch.from_numpy(plan.in_table(bases, B).reshape(-1)).to(storage.device)
        self.out_tbl = torch.from_numpy(plan.out_table(out.data_ptr(), B).reshape(-1)).to(storage.device)
        ids, off = plan.groups()
        self.ids = torch.from_numpy(ids).to(storage.device)
        self.off = off
        self.pos = torch.tensor(plan.key_of, dtype=torch.int32).to(storage.device)
        self.S = len(plan.stripes)

    def launch(self, stream=None, nstreams=8):
        X = self.X
        if self.S == 0:
            return
        if len(self.progs) == 1:
            X.xslp_encode_batch(self.progs[0], self.in_tbl, self.out_tbl, self.S, self.B, stream=stream)
        elif self.multi is not None:
            X.xslp_multi_decode(self.multi, self.pos, self.ids, self.off, self.in_tbl, self.out_tbl,
                                self.B, stream=stream)
        else:
            X.xslp_decode_batch_grouped(self.progs, self.ids, self.off, self.in_tbl, self.out_tbl,
                                        self.B, nstreams=nstreams, stream=stream)

    def close(self):
        for a in self.mapped:
            self.X.xslp_peer_close(a)
        self.mapped = []


def compile_plan(X, gf, plan, **kw):
    """One decode program per distinct (erased, survivors) key of the plan."""
    n, p = plan.pl.n, plan.pl.p
    bits = [X.xslp_decode_bitmatrix_from(gf, n, p, er, sv) for er, sv in plan.keys]
    return X.compile_many(bits, **kw) if bits else []


def fill_storage(X, placement, rank, storage, seed, enc_prog, chunk=64, stream=None):
    """Setup (untimed): this rank's blocks of the seeded codewords.  Data blocks come from the
    device generator (xslp_fill_random, keyed by global stripe and block), parity from the
    encode program; the blocks this rank owns are copied into storage [S][slots][B]."""
    import torch
    pl = placement
    n, p, B = pl.n, pl.p, storage.shape[-1]
    tmp = torch.empty((min(chunk, max(1, pl.stripes)), n + p, B), dtype=torch.uint8,
                      device=storage.device)
    for s0 in range(0, pl.stripes, chunk):
        c = min(chunk, pl.stripes - s0)
        X.xslp_fill_random(tmp, c, n + p, B, seed=seed, stripe0=s0, stream=stream)
        t = X.block_table(tmp, c, n + p, B).view(c, n + p)
        X.xslp_encode_batch(enc_prog, t[:, :n].contiguous(), t[:, n:].contiguous(), c, B,
                            stream=stream)
        for i in range(c):
            s = s0 + i
            for j in pl.blocks_of(rank, s):
                storage[s, pl.slot(s, j)].copy_(tmp[i, j])
    return storage
