"""BASELINE config 5: 8 k=20 subgraphs of 1,000,000 points each (config-2
distribution, d=128, 8M points), merged pairwise by S-Merge in a 3-level
tree (4 merges of 2M, 2 of 4M, 1 of 8M).  The reference runs the tree
serially on CPU (1,460 s).  Subgraphs are built untimed by this
package's NN-Descent.

* one GPU (default): the levels run one after another on one device;
* ``--dist`` under torchrun, one process per GPU (8 for config 5):
  ``python -m torch.distributed.run --nnodes=1 --nproc-per-node 8
  --master-addr 127.0.0.1 --master-port P tools/c5_tree.py --dist`` --
  ``distributed.tree_merge``: subgraph r on rank r, each level's merges
  sharded over their group's ranks through ``new_group`` sub-communicators
  (NCCL), groups of a level concurrent, no re-sharding between levels;
  per-level time = max over ranks of CUDA-event time.  With fewer GPUs than
  ranks (tests only) the ranks share cuda:0 over gloo.
Usage: python tools/c5_tree.py [--scale s] [--no-recall] [--dist]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main_dist(scale):
    """One rank of the 8-way tree (see the module docstring)."""
    import torch
    import torch.distributed as dist

    import paper_1908_00814_b200 as km
    from paper_1908_00814_b200 import distributed as D
    from paper_1908_00814_b200.engine import Engine

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    ngpu = torch.cuda.device_count()
    dev = rank if ngpu >= world else 0
    torch.cuda.set_device(dev)
    backend = "nccl" if ngpu >= world else "gloo"
    dist.init_process_group(backend)
    per = int(1_000_000 * scale)
    n = world * per
    t = time.perf_counter()
    ds = km.generate_int_gmm(n, 128, 1000, 20.0, seed=7)
    sets = [np.arange(r * per, (r + 1) * per, dtype=np.int64) for r in range(world)]
    eng = Engine(dev)
    mine = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=20), rank + 1, member_ids=sets[rank],
                         device=dev, out_device=True)
    groups = {tuple(m): dist.new_group(m) for _, m in D.tree_groups(world)}
    torch.cuda.synchronize()
    dist.barrier()
    setup = time.perf_counter() - t

    def group_comm(level, ranks):
        return D.TorchComm(groups[tuple(ranks)]) if rank in ranks else None

    marks = []

    def hook(level, members, cnt):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        marks.append((level, ev, cnt.count))

    params = km.MergeParams(k=20, seed=3)
    start = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    dist.barrier()
    start.record()
    final, log = D.tree_merge(ds, {rank: mine}, sets, params, world, group_comm, {rank: eng},
                              level_hook=hook)
    torch.cuda.synchronize()
    # per-level device times on this rank, then the max over ranks
    times, prev = [], start
    for level, ev, _ in marks:
        times.append(prev.elapsed_time(ev) / 1e3)
        prev = ev
    tt = torch.tensor(times, dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    evals = torch.tensor([sum(c for _, _, c in marks)], dtype=torch.float64,
                         device="cuda" if backend == "nccl" else "cpu")
    if rank == 0:
        print(f"c5 tree on {world} ranks ({backend}): n={n} setup {setup:.1f} s, level times (max over "
              f"ranks) {[round(x, 3) for x in tt.tolist()]} s, total {sum(tt.tolist()):.3f} s, "
              f"rank-0 evals {int(evals.item())}", flush=True)
    dist.destroy_process_group()


def main():
    if "--dist" in sys.argv:
        scale = float(sys.argv[sys.argv.index("--scale") + 1]) if "--scale" in sys.argv else 1.0
        return main_dist(scale)
    import torch
    import paper_1908_00814_b200 as km
    from configs_bench import recall

    scale = float(sys.argv[sys.argv.index("--scale") + 1]) if "--scale" in sys.argv else 1.0
    per = int(1_000_000 * scale)
    n = 8 * per
    t = time.perf_counter()
    ds = km.generate_int_gmm(n, 128, 1000, 20.0, seed=7)
    parts = [np.arange(i * per, (i + 1) * per, dtype=np.int64) for i in range(8)]
    graphs = [km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=20), i + 1, member_ids=p, out_device=True)
              for i, p in enumerate(parts)]
    torch.cuda.synchronize()
    print(f"setup: data + 8 subgraphs of {per} points in {time.perf_counter() - t:.1f} s", flush=True)
    params = km.MergeParams(k=20, seed=3)
    total_evals, level_times = 0, []
    t_all = time.perf_counter()
    level = graphs
    while len(level) > 1:
        t_l = time.perf_counter()
        nxt = []
        for a, b in zip(level[0::2], level[1::2]):
            c = km.DistanceCounter()
            nxt.append(km.s_merge(ds, a, b, params, counter=c, out_device=True))
            total_evals += c.count
        torch.cuda.synchronize()
        level_times.append(time.perf_counter() - t_l)
        level = nxt
    wall = time.perf_counter() - t_all
    out = level[0]
    rec = None
    if "--no-recall" not in sys.argv:
        host = km.KnnGraph(out.member_ids, out.k, out.metric)
        host.ids, host.dists, host.sizes = (out.ids.cpu().numpy(), out.dists.cpu().numpy(),
                                            out.sizes.cpu().numpy())
        rec = recall(ds, km.Metric.L2, host)
    print(f"c5 tree on 1 GPU: n={n} levels {[round(x, 3) for x in level_times]} s, total {wall:.3f} s, "
          f"evals {total_evals}, {total_evals / wall:.3e} evals/s, recall@10 {rec}", flush=True)


if __name__ == "__main__":
    main()
