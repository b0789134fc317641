"""CPU model of the reference-order slot layout used by the CUDA update
path (knnm_kernels.cuh: MembRec / partner_mask / pair_rank).

The reference applies a round's directed updates row by row in pair order
(u, p, q) (_kernels.py:217-254, 420-437).  The device writes each directed
update to slot  boff[row] + start(u, p_row) + rank(p_row, p_partner)  and
streams rows in slot order.  This test enumerates random neighbourhoods and
checks that the slot order equals the reference order for every row."""

import numpy as np
import pytest


def partner_mask(mode, cls):
    if mode == 0:
        return 0x3 if cls == 0 else 0x1
    if mode == 1:
        return {0: 0xC, 1: 0x4, 2: 0x3, 3: 0x1}[cls]
    return {0: 0xC, 1: 0x4, 2: 0xF, 3: 0x5}[cls]


def partner_self(mode, cls):
    return (mode == 0 and cls == 0) or (mode == 2 and cls == 2)


def admissible(na, nb, la, lb, mode):  # _kernels.py:391-399
    if not (na or nb):
        return False
    if mode == 1:
        return la != lb
    if mode == 2:
        return la != lb or (la == 1 and lb == 1)
    return True


@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("seed", range(6))
def test_slot_order_equals_reference_order(mode, seed):
    rng = np.random.default_rng(seed * 3 + mode)
    n = 40
    labels = rng.integers(0, 2, size=n) if mode else np.zeros(n, dtype=int)
    hoods = {}
    for u in range(n):
        w = int(rng.integers(0, 12))
        mem = np.sort(rng.choice(n, size=w, replace=False))
        new = rng.random(w) < 0.5
        hoods[u] = (mem, new)
    # reference order: for u, p<q admissible: (pa<-pb), (pb<-pa)
    ref = {r: [] for r in range(n)}
    for u in range(n):
        mem, new = hoods[u]
        for p in range(len(mem)):
            for q in range(p + 1, len(mem)):
                if admissible(new[p], new[q], labels[mem[p]], labels[mem[q]], mode):
                    ref[mem[p]].append((u, mem[q]))
                    ref[mem[q]].append((u, mem[p]))
    # slot model
    bound = np.zeros(n, dtype=int)
    memb = {r: [] for r in range(n)}
    info = {}
    for u in range(n):
        mem, new = hoods[u]
        cls = [(labels[m] != 0) * 2 + (0 if nw else 1) for m, nw in zip(mem, new)]
        cnt = [cls.count(c) for c in range(4)]
        P = np.zeros((4, len(mem) + 1), dtype=int)
        for c in range(4):
            P[c, 1:] = np.cumsum([x == c for x in cls])
        info[u] = (cls, P)
        for j, m in enumerate(mem):
            mk = partner_mask(mode, cls[j])
            part = sum(cnt[c] for c in range(4) if mk >> c & 1) - partner_self(mode, cls[j])
            if part > 0:
                bound[m] += part
                memb[m].append((u, j, part))
    start = {}
    for r in range(n):
        for (u, j, part) in memb[r]:
            start[(u, j)] = sum(p2 for (u2, _, p2) in memb[r] if u2 < u)
    got = {r: [None] * bound[r] for r in range(n)}
    for u in range(n):
        mem, new = hoods[u]
        cls, P = info[u]
        for p in range(len(mem)):
            for q in range(p + 1, len(mem)):
                if not admissible(new[p], new[q], labels[mem[p]], labels[mem[q]], mode):
                    continue
                for t, x in ((p, q), (q, p)):
                    mk = partner_mask(mode, cls[t])
                    rank = sum(P[c, x] for c in range(4) if mk >> c & 1)
                    if partner_self(mode, cls[t]) and t < x:
                        rank -= 1
                    slot = start[(u, t)] + rank
                    assert got[mem[t]][slot] is None, "slot collision"
                    got[mem[t]][slot] = (u, mem[x])
    for r in range(n):
        assert got[r] == ref[r]
