"""Dependency depth of the near graph at a BASELINE window (CPU analysis).

The coloured Gauss-Seidel sweep's result depends only on the visiting order of particles
that can interact in a round: pairs whose round-start gap is below 2 c_m (the near set).
With pi = (colour class, cell, slot), a particle can be decided once its near neighbours
that precede it in pi are decided.  This script measures, on a reference-prepared sample
of a configuration's window state, the degree of that graph and how many particles sit at
each dependency level (level 0 = no preceding near neighbour).

    python tools/near_graph_levels.py cfg4 [n]
"""
import os
import sys

import numpy as np
from scipy.spatial import cKDTree

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
    cfg = dict(bench.CONFIGS[name])
    if len(sys.argv) > 2:
        cfg["sample_n"] = int(sys.argv[2])
    _, S = bench.ref_sample_state(cfg, 20260101)
    pos, r, c_m, box = S["pos"], S["radii"], S["c_m"], float(S["Lb"][0])
    n, dim = pos.shape
    maxr = r.max()
    cell = 2.5 * maxr + c_m
    dims = max(3, int(np.floor(box / cell)))
    edge = box / dims
    cc = np.floor(pos / edge).astype(np.int64) % dims
    cutc = 2 * maxr + 3 * c_m
    s = 1
    while s * edge < cutc:
        s += 1
    m = s + 1
    body = m * (dims // m)
    col = np.where(cc < body, cc % m, m + cc - body)
    ncol = m + dims % m
    cls = col[:, 0] + ncol * (col[:, 1] + (ncol * col[:, 2] if dim == 3 else 0))
    key = cc[:, 0] + dims * (cc[:, 1] + (dims * cc[:, 2] if dim == 3 else 0))
    order = np.lexsort((np.arange(n), key, cls))  # pi: class, cell, slot
    rank = np.empty(n, np.int64)
    rank[order] = np.arange(n)
    tree = cKDTree(pos, boxsize=box)
    pairs = tree.query_pairs(2 * maxr + 2 * c_m, output_type="ndarray")
    d = pos[pairs[:, 0]] - pos[pairs[:, 1]]
    d -= box * np.round(d / box)
    keep = np.sqrt((d * d).sum(1)) <= r[pairs[:, 0]] + r[pairs[:, 1]] + 2 * c_m
    pairs = pairs[keep]
    print(f"{name}: n={n} dims={dims} classes={ncol ** dim} occupancy={n / dims ** dim:.2f} "
          f"near degree={2 * len(pairs) / n:.2f}")
    a, b = pairs[:, 0], pairs[:, 1]
    swap = rank[a] > rank[b]
    pred, succ = np.where(swap, b, a), np.where(swap, a, b)  # pred precedes succ
    level = np.zeros(n, np.int64)
    o = np.argsort(rank[succ])  # process edges by successor rank: predecessors final first
    for e in o:
        if level[succ[e]] < level[pred[e]] + 1:
            level[succ[e]] = level[pred[e]] + 1
    # the loop above needs all edges into pred handled first: true, since rank[pred] < rank[succ]
    # and edges are taken in increasing successor rank
    cnt = np.bincount(level)
    rem = n
    for k, c in enumerate(cnt):
        print(f"  level {k}: {c} ({100.0 * c / n:.2f}%)  pending before it: {rem}")
        rem -= c


if __name__ == "__main__":
    main()
