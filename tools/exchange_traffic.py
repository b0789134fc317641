"""Slot bytes the id-sharded exchange sends between ranks per config-2
merge, whole slot blocks vs written slots only (knnm_local_compact), at
world sizes P run as virtual ranks on one GPU (LoopbackComm).  Also checks
that every sharded result equals the single-GPU merge.
Usage: python tools/exchange_traffic.py [scale] [P ...]  -> JSON on stdout."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    import paper_1908_00814_b200 as km
    from paper_1908_00814_b200 import distributed as D
    from paper_1908_00814_b200.engine import Engine

    args = [a for a in sys.argv[1:]]
    scale = float(args[0]) if args else 1.0
    worlds = [int(a) for a in args[1:]] or [2, 4, 8]
    n = int(1_000_000 * scale)
    ds, s1, s2 = bench.make_inputs(km, n)
    g = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=20), 1, member_ids=s1)
    h = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=20), 2, member_ids=s2)
    mp = km.MergeParams(k=20, seed=3)
    want = km.s_merge(ds, g, h, mp)
    out = {"workload": f"config-2 S-Merge, n={n}, k=20, d=128", "worlds": {}}
    for P in worlds:
        engines = {r: Engine(0) for r in range(P)}
        row = {}
        for compact in (False, True):
            tr = {}
            t = time.perf_counter()
            got = D.s_merge_sharded(ds, g, h, mp, D.LoopbackComm(P), engines, compact=compact, traffic=tr)
            dt = time.perf_counter() - t
            same = bool(np.array_equal(got.ids, want.ids) and np.array_equal(got.dists, want.dists))
            row["compact" if compact else "blocks"] = {
                "remote_slot_bytes": int(sum(tr.values())),
                "per_rank_max_bytes": int(max(tr.values()) if tr else 0),
                "bit_identical": same, "loopback_wall_s": round(dt, 3)}
        row["reduction"] = row["blocks"]["remote_slot_bytes"] / max(row["compact"]["remote_slot_bytes"], 1)
        out["worlds"][P] = row
        for e in engines.values():
            e.close() if hasattr(e, "close") else None
        del engines
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
