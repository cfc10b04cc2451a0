"""Host-side model of the F2 fused exchange protocol (include/pft.h pft_comm_p2p_*):
G ranks run RO rounds; in round R = xround0 + it each rank pushes its shard's records into half
R & 1 of every rank's exchange buffer, adds 1 to its counter word in every rank's buffer, waits
until all of its own G counter words reach R + 1, then reads the whole half (P3).  Counters are
never reset; each rank stores its completed-round count (xround) for its next call.

The model runs the ranks as threads with adversarial delays and checks that every P3 read sees
exactly the round's records (no stale or overwritten slot) and that nothing deadlocks, across
calls with odd and even iteration counts and an early stop.  It also checks that the model is
sensitive: with per-call parity (it & 1 instead of the global round's), the adversarial schedule
exposes the overwrite race the kernel avoids."""
import random
import threading
import time

import pytest


class _Rank:
    def __init__(self, G, nrec):
        self.rec = [None] * nrec  # one buffer: half h occupies [h * stride, (h + 1) * stride)
        self.cnt = [0] * G
        self.xround = 0
        self.lock = threading.Lock()


def _run(G, K, calls, delay, global_parity=True, fixed_stride=True, timeout=5.0):
    """calls: executed-iteration counts per call, or (count, K_call) pairs (identical on every
    rank, as the stop decision is).  The exchange buffer holds 2 halves of G*ceil(K/G) records
    (K = the largest K_call); with fixed_stride=False a call uses its own G*ceil(K_call/G) stride.
    delay(rank, call, it, phase) -> seconds.  Returns the list of violations."""
    calls = [c if isinstance(c, tuple) else (c, K) for c in calls]
    kmax = max(kc for _, kc in calls)
    stride_max = G * -(-kmax // G)
    ranks = [_Rank(G, 2 * stride_max) for _ in range(G)]
    errors = []

    def worker(r):
        for ci, (n_exec, Kc) in enumerate(calls):
            kloc = -(-Kc // G)
            stride = stride_max if fixed_stride else G * kloc
            kb = r * kloc
            ks = max(0, min(Kc, kb + kloc) - kb)
            x0 = ranks[r].xround
            for it in range(n_exec):
                R = x0 + it
                time.sleep(delay(r, ci, it, "eval"))
                half = (R & 1) if global_parity else (it & 1)
                for q in range(G):
                    for j in range(ks):
                        ranks[q].rec[half * stride + kb + j] = (R, r, j)
                for q in range(G):
                    with ranks[q].lock:
                        ranks[q].cnt[r] += 1
                t0 = time.time()
                while min(ranks[r].cnt) < R + 1:
                    if time.time() - t0 > timeout:
                        errors.append(("timeout", r, ci, it))
                        return
                    time.sleep(1e-4)
                for src in range(G):
                    sb = src * kloc
                    for j in range(max(0, min(Kc, sb + kloc) - sb)):
                        time.sleep(delay(r, ci, it, "p3") / max(1, Kc))
                        got = ranks[r].rec[half * stride + sb + j]
                        if got != (R, src, j):
                            errors.append(("stale", r, ci, it, sb + j, got))
            ranks[r].xround = x0 + n_exec

    th = [threading.Thread(target=worker, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=60)
    assert not any(t.is_alive() for t in th), "deadlock"
    return errors


@pytest.mark.parametrize("G,K", [(2, 37), (3, 61), (8, 64), (8, 5)])
def test_protocol_random_delays(G, K):
    rng = random.Random(G * 1000 + K)
    lock = threading.Lock()

    def delay(r, ci, it, ph):
        with lock:
            return rng.random() * 2e-3
    # odd and even call lengths and a 1-iteration (early stop) call
    assert _run(G, K, [3, 1, 4, 2, 5], delay) == []


def test_protocol_adversarial_slow_reader():
    """Rank 1 lingers in P3 of the last round of a 1-iteration call while rank 0 races into the
    next call: global parity keeps rank 0's next push in the other half."""
    def delay(r, ci, it, ph):
        return 0.2 if (r == 1 and ci == 0 and ph == "p3") else 0.0
    assert _run(2, 16, [1, 2], delay) == []


def test_protocol_model_detects_per_call_parity():
    def delay(r, ci, it, ph):
        return 0.2 if (r == 1 and ci == 0 and ph == "p3") else 0.0
    errs = _run(2, 16, [1, 2], delay, global_parity=False)
    assert any(e[0] == "stale" for e in errs)


def test_protocol_varying_k_needs_fixed_stride():
    """Consecutive calls with different K (e.g. a schedule-length change): the half stride is fixed
    per buffer (include/pft.h, bench K), so round R's half never overlaps the other half a slow
    peer may still be reading; a per-call stride (G*ceil(K_call/G)) overlaps it."""
    def delay(r, ci, it, ph):
        return 0.3 if (r == 1 and ci == 0 and ph == "p3") else 0.0
    calls = [(1, 64), (2, 16)]
    assert _run(2, 64, calls, delay) == []
    errs = _run(2, 64, calls, delay, fixed_stride=False)
    assert any(e[0] == "stale" for e in errs)
