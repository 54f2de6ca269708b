"""CPU (gloo, world_size 2) checks of the 1D multi-GPU decomposition the NCCL path uses
(Alg. 1): ranks own rows [shard_begin(r), shard_begin(r+1)) (every rank
but the last owns ceil(n/P) rows, so labels allgather in place into a P*B buffer), compute E for
their rows, reduce (k+1) fp64 partials by allgather + fixed-order sum, assign locally, and
allgather the labels. The per-rank arithmetic here is the oracle's; what is under test is the
shard layout of libkkm (kkm_shard_begin) and the exchange schedule, against the 1-rank oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def shard_begin(n, r, P):
    import paper_2601_17136_b200 as kkm  # the library's own layout function (pure, no CUDA)
    return kkm.shard_begin(n, r, P)


def one_iteration_ranked(X, labels, k, args, P, rank, allgather):
    """The exchange schedule of one 1D iteration, as rank `rank` of P executes it."""
    n = X.shape[0]
    B = -(-n // P)
    r0, r1 = shard_begin(n, rank, P), shard_begin(n, rank + 1, P)
    assert r0 == min(n, rank * B) and r1 - r0 <= B
    rows = np.arange(r0, r1)
    Kr = oracle.kernel_rows(X, rows, *args) if rows.size else np.zeros((0, n))
    diag = oracle.kernel_diag(X, *args, rows=rows) if rows.size else np.zeros(0)
    sizes = np.bincount(labels, minlength=k)
    E = oracle.E_rows(Kr, labels, k) if rows.size else np.zeros((0, k))
    # local partials: sum_{i in L_c, i local} z_i (c < k) and sum_i (K_ii - z_i) (slot k)
    part = np.zeros(k + 1)
    for ii, i in enumerate(rows):
        z = E[ii, labels[i]]
        part[labels[i]] += z
        part[k] += diag[ii] - z
    allp = allgather(part)                                 # P x (k+1)
    tot = np.zeros(k + 1)
    for r in range(P):                                     # fixed rank order
        tot += allp[r]
    cn = np.where(sizes > 0, tot[:k] / np.maximum(sizes, 1), np.inf)
    J = tot[k]
    new_local, _ = oracle.assign(E, diag, cn) if rows.size else (np.zeros(0, np.int32), None)
    send = np.full(B, -1, dtype=np.int32)
    send[:new_local.size] = new_local
    gathered = allgather(send).reshape(-1)[:n]             # in place: rank r at offset r*B
    return gathered, cn, J


def _worker(rank, P, port, n, k, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=P)

    def allgather(a):
        t = torch.from_numpy(np.ascontiguousarray(a))
        out = [torch.empty_like(t) for _ in range(P)]
        dist.all_gather(out, t)
        return np.stack([o.numpy() for o in out])

    X, cfg = synth.make_config("har200k", n=n)
    args = (cfg["kind"], cfg["gamma"], cfg["coef0"], cfg["degree"])
    labels = oracle.round_robin(n, k)
    res = []
    for _ in range(3):
        labels, cn, J = one_iteration_ranked(X, labels, k, args, P, rank, allgather)
        res.append((labels.copy(), cn, J))
    q.put((rank, res))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n", [301, 300])
def test_gloo_world2_matches_single_rank(n):
    P, k = 2, 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, P, port, n, k, q)) for r in range(P)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(P))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    X, cfg = synth.make_config("har200k", n=n)
    ref = oracle.fit(X, k, cfg["kind"], cfg["gamma"], max_iter=3, keep_trace=True)
    for t in range(3):
        lab0, cn0, J0 = out[0][t]
        lab1, cn1, J1 = out[1][t]
        assert np.array_equal(lab0, lab1)                   # every rank holds the same labels
        assert np.array_equal(cn0, cn1) and J0 == J1        # bitwise-identical c and J
        assert np.array_equal(lab0, ref["label_trace"][t + 1])
        assert abs(J0 - ref["J_trace"][t]) <= 1e-12 * abs(ref["J_trace"][t])


class _Rendezvous:
    """In-process stand-in for the collectives: every simulated rank deposits its buffer for
    collective #t; the call returns the stacked buffers once all P have arrived."""

    def __init__(self, P):
        self.P, self.slots = P, {}

    def rank_view(self, rank):
        counter = [0]

        def allgather(a):
            t = counter[0]
            counter[0] += 1
            self.slots.setdefault(t, {})[rank] = np.array(a)
            if len(self.slots[t]) < self.P:
                raise _Pending(t)
            return np.stack([self.slots[t][r] for r in range(self.P)])
        return allgather


class _Pending(Exception):
    pass


@pytest.mark.parametrize("n,P", [(5, 4), (37, 3), (64, 8), (10, 1)])
def test_shard_layout_in_process(n, P):
    """Ragged shards, including an empty last rank (n=5, P=4), simulated in one process by
    re-running each rank's program until all of its collectives have completed."""
    X = synth.blobs(n, 3, 2, seed=n)
    k = 2
    args = (oracle.LINEAR, 1.0, 0.0, 1)
    labels = oracle.round_robin(n, k)
    rv = _Rendezvous(P)
    results = {}
    for _ in range(3):  # two collectives per iteration -> at most 3 sweeps
        for r in range(P):
            if r in results:
                continue
            try:
                results[r] = one_iteration_ranked(X, labels, k, args, P, r, rv.rank_view(r))
            except _Pending:
                pass
    assert len(results) == P
    ref = oracle.iteration(oracle.kernel_matrix(X, *args), oracle.kernel_diag(X, *args), labels, k)
    for lab, cn, J in results.values():
        assert np.array_equal(lab, ref["new_labels"])
        assert np.allclose(cn, ref["cnorm"], rtol=1e-13)
        assert abs(J - ref["J"]) <= 1e-12 * max(1.0, abs(ref["J"]))
    b = [shard_begin(n, r, P) for r in range(P + 1)]
    assert b[0] == 0 and b[-1] == n and all(x <= y for x, y in zip(b, b[1:]))


def one_iteration_15d(X, labels, k, args, pr, pc, rank, coll):
    """One iteration of the 1.5D schedule (Alg. 2) as rank = gi + gj * pr of a pr x pc
    grid executes it: partial E for the points of column block gj against row block gi, a
    column-split reduce-scatter over process column gj, then the 1D tail."""
    n = X.shape[0]
    P = pr * pc
    B = -(-n // P)
    gi, gj = rank % pr, rank // pr
    a0, a1 = min(n, gj * pr * B), min(n, (gj + 1) * pr * B)   # column block gj (A set)
    b0, b1 = min(n, gi * pc * B), min(n, (gi + 1) * pc * B)   # row block gi (B set)
    sizes = np.bincount(labels, minlength=k)
    Ka = oracle.kernel_rows(X, np.arange(a0, a1), *args)[:, b0:b1] if a1 > a0 else np.zeros((0, b1 - b0))
    lb = labels[b0:b1]
    Spart = np.zeros((pr * B, k))
    for c in range(k):
        Spart[:a1 - a0, c] = Ka[:, lb == c].sum(axis=1)         # sum over the B set only
    # reduce-scatter along process column gj: rank (l, gj) keeps rows [l B, (l+1) B)
    allS = coll("col", gj, gi, Spart)                          # pr x (pr B) x k from column peers
    mine = sum(allS[l] for l in range(pr))[gi * B:(gi + 1) * B]
    r0, r1 = min(n, rank * B), min(n, (rank + 1) * B)
    assert r0 == a0 + gi * B or r0 == n
    E = mine[:r1 - r0] / np.maximum(sizes, 1)
    diag = oracle.kernel_diag(X, *args, rows=np.arange(r0, r1)) if r1 > r0 else np.zeros(0)
    part = np.zeros(k + 1)
    for ii, i in enumerate(range(r0, r1)):
        z = E[ii, labels[i]]
        part[labels[i]] += z
        part[k] += diag[ii] - z
    allp = coll("world", 0, rank, part)
    tot = np.zeros(k + 1)
    for r in range(P):
        tot += allp[r]
    cn = np.where(sizes > 0, tot[:k] / np.maximum(sizes, 1), np.inf)
    new_local, _ = oracle.assign(E, diag, cn) if r1 > r0 else (np.zeros(0, np.int32), None)
    send = np.full(B, -1, dtype=np.int32)
    send[:new_local.size] = new_local
    return coll("world", 1, rank, send).reshape(-1)[:n], cn, tot[k]


class _GroupRendezvous:
    """In-process collectives over named groups: ("col", j) has the pr ranks of process column j
    ordered by process row; ("world", tag) all ranks."""

    def __init__(self, pr, pc):
        self.pr, self.pc, self.slots = pr, pc, {}

    def view(self, rank):
        counter = {}

        def coll(group, tag, member, buf):
            key = (group, tag, counter.get((group, tag), 0))
            counter[(group, tag)] = key[2] + 1
            size = self.pr if group == "col" else self.pr * self.pc
            self.slots.setdefault(key, {})[member] = np.array(buf)
            if len(self.slots[key]) < size:
                raise _Pending(key)
            return np.stack([self.slots[key][m] for m in range(size)])
        return coll


@pytest.mark.parametrize("n,pr,pc", [(64, 2, 2), (101, 2, 4), (37, 3, 2), (50, 4, 1), (9, 2, 2)])
def test_15d_schedule_matches_oracle(n, pr, pc):
    X = synth.blobs(n, 3, 3, seed=n + pr)
    k = 3
    args = (oracle.POLY, 0.5, 1.0, 2)
    labels = oracle.round_robin(n, k)
    rv = _GroupRendezvous(pr, pc)
    results = {}
    for _ in range(4):
        for r in range(pr * pc):
            if r in results:
                continue
            try:
                results[r] = one_iteration_15d(X, labels, k, args, pr, pc, r, rv.view(r))
            except _Pending:
                pass
    assert len(results) == pr * pc
    ref = oracle.iteration(oracle.kernel_matrix(X, *args), oracle.kernel_diag(X, *args), labels, k)
    for lab, cn, J in results.values():
        assert np.array_equal(lab, ref["new_labels"])
        assert np.allclose(cn, ref["cnorm"], rtol=1e-12)
        assert abs(J - ref["J"]) <= 1e-10 * max(1.0, abs(ref["J"]))


# ---- the default 1D f1 exchange: each rank's S contributions from the library's own
# plan (kkm_plan_query pieces: row parts + mirrored column parts), summed over the ranks as int64
# fixed point by a real allreduce (gloo), then a3/a4 replicated on every rank -- and the opt-in
# distributed variant (KKM_LSA=1): each rank finishes only its own rows, exchanges its (k + 1)
# partials, and the labels are gathered. The arithmetic per rank is the oracle's.
FX = 2.0 ** 40  # fixed-point scale (|S| * 2^40 << 2^63 at these sizes)


def f1_contrib(pcs, K, labels, k):
    n = K.shape[0]
    V = np.zeros((n, k))
    V[np.arange(n), labels] = 1.0
    Sr = np.zeros((n, k))
    for r0, nr, c0, nc, cd in pcs:
        Sr[r0:r0 + nr] += K[r0:r0 + nr, c0:c0 + nc] @ V[c0:c0 + nc]
        if cd < c0 + nc:
            a = max(cd, c0)
            Sr[a:c0 + nc] += K[r0:r0 + nr, a:c0 + nc].T @ V[r0:r0 + nr]
    return np.rint(Sr * FX).astype(np.int64)


def _worker_f1(rank, P, port, n, k, distributed, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=P)
    import paper_2601_17136_b200 as kkm
    X, cfg = synth.make_config("har200k", n=n)
    args = (cfg["kind"], cfg["gamma"], cfg["coef0"], cfg["degree"])
    K = oracle.kernel_matrix(X, *args)
    diag = np.diag(K).copy()
    p = kkm.default_params()
    p.k, p.kind, p.path, p.symmetric, p.kstore = k, kkm.KERNEL_GAUSSIAN, kkm.PATH_MATERIALIZE, kkm.SYM_ON, kkm.KSTORE_FP16X2
    info, pcs = kkm.plan_query(p, n, X.shape[1], rank=rank, nranks=P)
    assert info.exchange == kkm.XCHG_S_ALLREDUCE
    labels = oracle.round_robin(n, k)
    res = []
    for _ in range(3):
        S = torch.from_numpy(f1_contrib(pcs, K, labels, k))
        dist.all_reduce(S)  # exact integer sum: the same bits on every rank, any order
        sizes = np.bincount(labels, minlength=k)
        E = (S.numpy().astype(np.float64) / FX) / np.maximum(sizes, 1)
        if not distributed:  # replicated a3/a4 over all points
            cn = oracle.cnorm(E, labels, k)
            J = oracle.objective(diag, labels, k, cn)
            labels, _ = oracle.assign(E, diag, cn)
        else:  # own rows only; (k + 1) partials gathered and summed in rank order; labels gathered
            r0, r1 = shard_begin(n, rank, P), shard_begin(n, rank + 1, P)
            part = np.zeros(k + 1)
            for i in range(r0, r1):
                part[labels[i]] += E[i, labels[i]]
                part[k] += diag[i] - E[i, labels[i]]
            allp = [torch.zeros(k + 1, dtype=torch.float64) for _ in range(P)]
            dist.all_gather(allp, torch.from_numpy(part))
            tot = np.zeros(k + 1)
            for r in range(P):
                tot += allp[r].numpy()
            cn = np.where(sizes > 0, tot[:k] / np.maximum(sizes, 1), np.inf)
            J = tot[k]
            mine, _ = oracle.assign(E[r0:r1], diag[r0:r1], cn)
            B = -(-n // P)
            send = torch.full((B,), -1, dtype=torch.int32)
            send[:mine.size] = torch.from_numpy(mine.astype(np.int32))
            out = [torch.empty(B, dtype=torch.int32) for _ in range(P)]
            dist.all_gather(out, send)
            labels = torch.cat(out).numpy()[:n]
        res.append((np.asarray(labels).copy(), np.asarray(cn), float(J)))
    q.put((rank, res))
    dist.destroy_process_group()


@pytest.mark.parametrize("distributed", [False, True], ids=["replicated", "distributed"])
def test_gloo_world2_f1_exchange_matches_oracle(distributed):
    P, k, n = 2, 6, 3001
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_f1, args=(r, P, port, n, k, distributed, q)) for r in range(P)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in range(P))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    X, cfg = synth.make_config("har200k", n=n)
    ref = oracle.fit(X, k, cfg["kind"], cfg["gamma"], max_iter=3, keep_trace=True)
    for t in range(3):
        lab0, cn0, J0 = out[0][t]
        lab1, cn1, J1 = out[1][t]
        assert np.array_equal(lab0, lab1)
        assert np.array_equal(cn0, cn1) and J0 == J1  # bitwise the same on both ranks
        assert np.array_equal(lab0, ref["label_trace"][t + 1])
        assert abs(J0 - ref["J_trace"][t]) <= 1e-9 * abs(ref["J_trace"][t])
