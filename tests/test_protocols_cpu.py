"""CPU emulation of the two peer-memory protocols of the multi-GPU path at
world size 8 (the CUDA kernels cannot run here; these check the protocol
design -- sequence numbers, flags, buffer reuse -- under adversarial
scheduling, with one thread per rank and random delays between every step).

1. The owner-side push pre-gather (hg_peer.cu hg_pregather_push_multi):
   mark own request list -> signal flags[rank] = seq in every peer's mailbox
   -> wait for every peer's flag -> serve: copy the rows homed here into every
   requester's staging -> signal done -> wait for every peer's done -> the
   requester's gather reads its staging.  Invariants: every staged row is the
   row the requester asked for in THIS call (no stale or torn rows), and no
   request list changes while a peer is serving it.
2. The NVLink gradient all-reduce (hg_p2p_allreduce): push this rank's vector
   into slot [rank] of buffer (seq & 1) of every peer, signal, wait, sum.
   Invariant: every rank's sum equals the true sum at every step, with only
   two buffers.
"""
import random
import threading
import time

import numpy as np

S = 8


def _jitter(rng):
    if rng.random() < 0.3:
        time.sleep(rng.random() * 2e-4)


def _wait(cond, what):
    t0 = time.time()
    while not cond():
        if time.time() - t0 > 20:
            raise AssertionError(f"protocol deadlock waiting for {what}")
        time.sleep(0)


def test_push_pregather_handshake_world8():
    calls = 12
    n = 4000
    home = np.random.default_rng(0).integers(0, S, n)
    row = lambda v, call: v * 1000 + call  # noqa: E731  (the owner's value at that call)
    flags = np.zeros((S, S), dtype=np.int64)     # flags[box][peer]
    done = np.zeros((S, S), dtype=np.int64)
    lists = [[] for _ in range(S)]               # request list in each rank's mailbox
    staging = [dict() for _ in range(S)]
    serving = np.zeros(S, dtype=np.int64)        # peers currently reading rank r's list
    lock = threading.Lock()
    errors = []

    def rank_main(r):
        rng = random.Random(r)
        wants = np.random.default_rng(100 + r)
        try:
            for seq in range(1, calls + 1):
                # mark: this call's remote vertices (nobody may be serving our list now)
                with lock:
                    assert serving[r] == 0, "request list rewritten while a peer serves it"
                req = sorted(set(int(v) for v in wants.integers(0, n, 300) if home[v] != r))
                lists[r] = req
                staging[r] = {}
                _jitter(rng)
                for p in range(S):               # signal requests
                    if p != r:
                        flags[p][r] = seq
                _wait(lambda: all(flags[r][p] >= seq for p in range(S) if p != r), "requests")
                for p in range(S):               # serve every peer's rows homed here
                    if p == r:
                        continue
                    with lock:
                        serving[p] += 1
                    for v in list(lists[p]):
                        if home[v] == r:
                            staging[p][v] = row(v, seq)
                        if rng.random() < 0.01:
                            _jitter(rng)
                    with lock:
                        serving[p] -= 1
                for p in range(S):               # signal done
                    if p != r:
                        done[p][r] = seq
                _wait(lambda: all(done[r][p] >= seq for p in range(S) if p != r), "rows")
                for v in req:                    # the gather reads the staged rows
                    if staging[r].get(v) != row(v, seq):
                        raise AssertionError(f"rank {r} call {seq}: row {v} stale or missing")
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(S)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors[0]


def test_p2p_allreduce_double_buffer_world8():
    steps, n = 40, 64
    bufs = np.zeros((S, 2, S, n))                # receiver x parity x sender x n
    flags = np.zeros((S, S), dtype=np.int64)
    seqs = [0] * S
    errors = []

    def grad(r, s):
        return np.random.default_rng(r * 1000 + s).standard_normal(n)

    def rank_main(r):
        rng = random.Random(r)
        try:
            for step in range(1, steps + 1):
                g = grad(r, step)
                s = seqs[r] + 1
                par = s & 1
                for p in range(S):               # push into every peer's slot [r]
                    if p != r:
                        bufs[p, par, r] = g
                        _jitter(rng)
                seqs[r] = s
                for p in range(S):               # signal
                    if p != r:
                        flags[p][r] = s
                _wait(lambda: all(flags[r][p] >= s for p in range(S) if p != r), "grads")
                total = g + sum(bufs[r, par, p] for p in range(S) if p != r)
                want = sum(grad(q, step) for q in range(S))
                if not np.allclose(total, want):
                    raise AssertionError(f"rank {r} step {step}: wrong sum (buffer reused early)")
                _jitter(rng)
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(S)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors[0]
