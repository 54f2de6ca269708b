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
