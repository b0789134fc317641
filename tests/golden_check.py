"""Shared golden-vector harness: rebuild a case's inputs and compare a
merge implementation (oracle or CUDA path) with tests/golden/golden.json."""

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import cases as C  # noqa: E402

with open(os.path.join(HERE, "golden", "golden.json")) as f:
    GOLDEN = json.load(f)


def h_graph(ids, dists, sizes) -> str:
    h = hashlib.sha256()
    for a in (np.ascontiguousarray(ids, dtype=np.int32), np.ascontiguousarray(dists, dtype=np.float64),
              np.ascontiguousarray(sizes, dtype=np.int32)):
        h.update(a.tobytes())
    return h.hexdigest()


def report_list(rep):
    return [[r.iteration, r.pairs, r.updates, r.phi, r.distance_count] for r in rep.rounds]


def inputs(oracle, name):
    """(vectors, g, h, s1, s2) for a case, subgraphs built by the oracle
    (pinned against the reference's own hashes by the caller)."""
    spec = GOLDEN["cases"][name]["spec"]
    vec = C.make_data(spec)
    s1, s2 = C.split(spec)
    k, metric = spec["k"], spec["metric"]
    if spec["op"] == "nnd":
        return vec, None, None, s1, s2
    if spec.get("inputs") == "bruteforce":
        g = oracle.brute_force_graph(vec, metric, k, member_ids=s1)
        h = (oracle.brute_force_graph(vec, metric, k, member_ids=s2) if len(s2) > k
             else oracle.OGraph(s2, k, metric))
    else:
        g, _, _ = oracle.nn_descent(vec, metric, k, spec["g_seed"], member_ids=s1)
        h = (oracle.nn_descent(vec, metric, k, spec["h_seed"], member_ids=s2)[0]
             if spec["op"] == "smerge" else None)
    return vec, g, h, s1, s2
