"""Generate golden vectors from the REFERENCE implementation (knnmerge).

Run in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It writes tests/golden/golden.json.  For every case it records, from the
reference itself: the sha256 of the input subgraphs (built by the
reference's nn_descent), the sha256 of the merged graph (ids, dists, sizes),
the distance count, the BuildReport (phi_initial, per-round pairs / updates
/ phi / distance_count, converged) and the per-round end-of-round state hash
(ids, dists, flags, sizes in local index space) captured through a shim on
knnmerge._kernels.reverse_csr (first call of every round,
construct.py:138) -- the replay contract of SURVEY.md §6.3.  Small cases
also store full output arrays.

Inputs are regenerated from seeds by tests/golden/cases.py on both sides, so
the fixture is small and contains no dataset.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import cases as C  # noqa: E402


def h_graph(ids, dists, sizes) -> str:
    h = hashlib.sha256()
    for a in (np.ascontiguousarray(ids, dtype=np.int32), np.ascontiguousarray(dists, dtype=np.float64),
              np.ascontiguousarray(sizes, dtype=np.int32)):
        h.update(a.tobytes())
    return h.hexdigest()


def h_state(ids, dists, flags, sizes) -> str:
    h = hashlib.sha256()
    for a in (np.ascontiguousarray(ids, dtype=np.int32), np.ascontiguousarray(dists, dtype=np.float64),
              np.ascontiguousarray(flags, dtype=np.uint8), np.ascontiguousarray(sizes, dtype=np.int32)):
        h.update(a.tobytes())
    return h.hexdigest()[:32]


class RoundShim:
    """Capture end-of-round state hashes from the reference's round engine."""

    def __init__(self, km):
        self.km = km
        self.k = km._kernels
        self.states = []
        self._arrays = None

    def __enter__(self):
        shim = self
        orig_rev = self.k.reverse_csr
        orig_rounds = self.km.merge._descent_rounds
        orig_rounds_c = self.km.construct._descent_rounds

        def rev(ids, flags, sizes):
            if shim._arrays is not None and shim._started:
                a = shim._arrays
                shim.states.append(h_state(a[0], a[1], a[2], a[3]))
            shim._started = True
            return orig_rev(ids, flags, sizes)

        def rounds_wrap(orig):
            def f(sub, metric, ids, dists, flags, sizes, *rest, **kw):
                shim._arrays = (ids, dists, flags, sizes)
                shim._started = False
                out = orig(sub, metric, ids, dists, flags, sizes, *rest, **kw)
                shim.states.append(h_state(ids, dists, flags, sizes))
                shim._arrays = None
                return out
            return f

        self._saved = (orig_rev, orig_rounds, orig_rounds_c)
        self.k.reverse_csr = rev
        self.km.merge._descent_rounds = rounds_wrap(orig_rounds)
        self.km.construct._descent_rounds = rounds_wrap(orig_rounds_c)
        return self

    def __exit__(self, *a):
        orig_rev, orig_rounds, orig_rounds_c = self._saved
        self.k.reverse_csr = orig_rev
        self.km.merge._descent_rounds = orig_rounds
        self.km.construct._descent_rounds = orig_rounds_c


def report_dict(rep) -> dict:
    return {
        "phi_initial": rep.phi_initial,
        "converged": bool(rep.converged),
        "rounds": [[r.iteration, r.pairs, r.updates, r.phi, r.distance_count] for r in rep.rounds],
    }


def main():
    import knnmerge as km

    out = {"reference": "knnmerge (pkg/src/knnmerge) via PYTHONPATH=/root/reference/pkg/src",
           "numpy": np.__version__, "cases": {}}
    for name, spec in C.CASES.items():
        vectors = C.make_data(spec)
        ds = km.Dataset.from_dense(vectors, validate=False)
        metric = km.Metric(spec["metric"])
        k = spec["k"]
        s1, s2 = C.split(spec)
        rec = {"spec": spec}
        if spec["op"] == "nnd":
            with RoundShim(km) as sh:
                c = km.DistanceCounter()
                g, rep = km.nn_descent(ds, metric, km.DescentParams(k=k, **spec.get("dp", {})),
                                       spec["g_seed"], member_ids=s1, counter=c, return_report=True)
            rec.update(out=h_graph(g.ids, g.dists, g.sizes), count=c.count,
                       report=report_dict(rep), states=sh.states)
        else:
            if spec.get("inputs") == "bruteforce":
                g = km.brute_force_graph(ds, metric, k, member_ids=s1)
                h = (km.brute_force_graph(ds, metric, k, member_ids=s2) if len(s2) > k
                     else km.KnnGraph(s2, k, metric))
            else:
                dp = km.DescentParams(k=k)
                g = km.nn_descent(ds, metric, dp, spec["g_seed"], member_ids=s1)
                h = km.nn_descent(ds, metric, dp, spec["h_seed"], member_ids=s2)
            rec["g"] = h_graph(g.ids, g.dists, g.sizes)
            mp = km.MergeParams(k=k, seed=spec["merge_seed"], **spec.get("mp", {}))
            with RoundShim(km) as sh:
                c = km.DistanceCounter()
                if spec["op"] == "smerge":
                    rec["h"] = h_graph(h.ids, h.dists, h.sizes)
                    u, rep = km.s_merge(ds, g, h, mp, counter=c, return_report=True)
                else:
                    raw = s2 if spec.get("raw", "s2") == "s2" else np.array([], dtype=np.int64)
                    u, rep = km.j_merge(ds, g, raw, mp, counter=c, return_report=True)
            rec.update(out=h_graph(u.ids, u.dists, u.sizes), count=c.count,
                       report=report_dict(rep), states=sh.states)
            if u.n <= 64:
                rec["arrays"] = {"ids": u.ids.tolist(), "dists": u.dists.tolist(),
                                 "sizes": u.sizes.tolist()}
        out["cases"][name] = rec
        print(name, rec["out"][:16], rec.get("count"), len(rec.get("states", [])), flush=True)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__" and "--extra" not in sys.argv:
    main()


def extra():
    """H-Merge and KNNG file golden vectors (tests/golden/golden_extra.json)."""
    import knnmerge as km
    import knnmerge.io as kio
    import tempfile

    out = {}
    ds = km.Dataset.from_dense(C.make_data(dict(data="uniform", n=2000, d=4, data_seed=13)), validate=False)
    c = km.DistanceCounter()
    graph, hier, reps = km.h_merge(ds, km.Metric.L2, km.MergeParams(k=10, seed=4), counter=c,
                                   return_report=True)
    out["hmerge"] = dict(out=h_graph(graph.ids, graph.dists, graph.sizes), count=c.count,
                         layer_sizes=hier.layer_sizes,
                         layers=[h_graph(l.graph.ids, l.graph.dists, l.graph.sizes) for l in hier.layers],
                         reports=[[name, report_dict(r)] for name, r in reps])
    # the same build with layer snapshots on disk: every file's hash
    # (reference merge.py:457-467 _maybe_snapshot, io.py:201-248)
    import hashlib
    import tempfile

    with tempfile.TemporaryDirectory() as tmp:
        km.h_merge(ds, km.Metric.L2, km.MergeParams(k=10, seed=4), snapshot_dir=tmp)
        out["hmerge"]["snapshot_sha256"] = {
            f: hashlib.sha256(open(os.path.join(tmp, f), "rb").read()).hexdigest()
            for f in sorted(os.listdir(tmp))}
    ds2 = km.Dataset.from_dense(C.make_data(dict(data="uniform", n=300, d=5, data_seed=2)), validate=False)
    g = km.nn_descent(ds2, km.Metric.L2, km.DescentParams(k=6), 3, member_ids=np.arange(0, 300, 2))
    with tempfile.TemporaryDirectory() as tmp:
        kio.save_graph(tmp + "/g.knng", g)
        kio.save_member_ids(tmp + "/g.ids", g.member_ids)
        import hashlib
        out["knng"] = dict(graph=h_graph(g.ids, g.dists, g.sizes),
                           file_sha256=hashlib.sha256(open(tmp + "/g.knng", "rb").read()).hexdigest(),
                           ids_sha256=hashlib.sha256(open(tmp + "/g.ids", "rb").read()).hexdigest())
    with open(os.path.join(HERE, "golden_extra.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("extra", out["hmerge"]["layer_sizes"], out["hmerge"]["count"])


if __name__ == "__main__" and "--extra" in sys.argv:
    extra()
