"""Regenerate the committed golden fixtures (run in the dev container, where
/root/reference exists and oracle/_ref/libmgraph_ref.so is built from it).

  python tests/golden/make_golden.py

Writes
  tests/golden/reference_pins.json  known answers quoted from the reference's own
                                    unit tests (file:line recorded per entry)
  tests/golden/ref_vectors.npz      outputs of the UNMODIFIED reference (engine +
                                    sequential oracles) on small graphs, with the
                                    graphs themselves, so the GPU box can check
                                    parity without /root/reference.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402

T = "/root/reference/proj/tests/"

PINS = {
    "bfs_p4_two_way": {
        "cite": T + "test_engine.cpp:250-260,289-295; test_primitives.cpp:41-44",
        "graph": "p4", "owner": [0, 0, 1, 1], "source": 0,
        "labels": [0, 1, 2, 3], "supersteps": 4, "h_total": 2,
        "h_matrix": [[0, 1], [1, 0]], "combine_ops": 2,
    },
    "sssp_p4_weighted": {
        "cite": T + "test_primitives.cpp:195-202",
        "edges": [[0, 1, 2], [1, 2, 3], [2, 3, 1]], "nv": 4, "owner": [0, 0, 1, 1],
        "source": 0, "dists": [0, 2, 5, 6],
    },
    "cc_triangle_isolated": {
        "cite": T + "test_primitives.cpp:243-249",
        "edges": [[0, 1], [1, 2], [0, 2]], "nv": 4, "components": [0, 0, 0, 3],
    },
    "cc_edgeless": {
        "cite": T + "test_primitives.cpp:251-255", "nv": 5, "components": [0, 1, 2, 3, 4],
    },
    "bc_p4": {
        "cite": T + "test_primitives.cpp:281-287", "graph": "p4", "owner": [0, 0, 1, 1],
        "source": 0, "bc": [0, 2, 1, 0],
    },
    "bc_star5_leaf": {
        "cite": T + "test_primitives.cpp:289-295",
        "edges": [[0, 1], [0, 2], [0, 3], [0, 4]], "nv": 5, "source": 1, "bc_center": 3.0,
    },
    "pr_single_vertex": {
        "cite": T + "test_primitives.cpp:319-323", "nv": 1, "rank": 1.0,
    },
    "direction_rule_table": {
        "cite": T + "test_primitives.cpp:102-150 (also acceptance.cpp:336-384)",
        # (current 0=F/1=B, fv, bv, do_a, do_b, switched, expect)
        "cases": [
            [0, 1000, 5000, 0.01, 0.1, 0, 1], [1, 100, 5000, 0.01, 0.1, 0, 0],
            [0, 1000, 5000, 0.01, 0.1, 1, 0], [0, 1e9, 1, 0.01, 0.1, 1, 0],
            [0, 50, 5000, 0.01, 0.1, 0, 0], [0, 50.0001, 5000, 0.01, 0.1, 0, 1],
            [0, 1, 1e6, 0.01, 0.1, 0, 0], [0, 0, 0, 0.01, 0.1, 0, 0],
            [1, 500, 5000, 0.01, 0.1, 0, 1], [1, 499.999, 5000, 0.01, 0.1, 0, 0],
            [1, 0, 0, 0.01, 0.1, 0, 1], [1, 1e9, 1e6, 0.01, 0.1, 1, 1],
            [0, 10, 100, 0.5, 0.9, 0, 0], [0, 51, 100, 0.5, 0.9, 0, 1],
            [1, 89, 100, 0.5, 0.9, 0, 0], [1, 91, 100, 0.5, 0.9, 0, 1],
            [0, 100, 100, 1.0, 1.0, 0, 0], [0, 101, 100, 1.0, 1.0, 0, 1],
            [1, 99, 100, 1.0, 1.0, 0, 0], [1, 100, 100, 1.0, 1.0, 0, 1],
        ],
    },
    "direction_estimates": {
        "cite": T + "test_primitives.cpp:152-157",
        "args": [10, 900, 100, 5000, 1000], "fv": 50.0, "bv": 9000.0,
    },
    "partition_p4_two_way": {
        "cite": T + "test_partition.cpp:96-129 (borders of the P4 split)",
        "owner": [0, 0, 1, 1], "borders_01": [2], "borders_10": [1],
    },
}


def main():
    with open(os.path.join(HERE, "reference_pins.json"), "w") as f:
        json.dump(PINS, f, indent=1)

    vec = {}
    # RMAT(12,16,1): fixtures::rmat (tests/fixtures.hpp:56-63) — test_primitives BFS/SSSP/CC pins
    g = ref.RefGraph.rmat(12, 16, 1)
    off, col, _ = g.arrays()
    vec["rmat12_off"], vec["rmat12_col"] = off, col
    vec["rmat12_bfs0"] = g.seq_bfs(0)
    vec["rmat12_cc"] = g.seq_cc()
    gw = g.weighted(0, 64, 2)  # fixtures::rmat(..., weights=true): seed+1
    vec["rmat12_w"] = gw.arrays()[2]
    vec["rmat12_dijkstra0"] = gw.seq_dijkstra(0)
    # RMAT(10,8,12): BC pin graph (test_primitives.cpp:297-308), source 1
    g10 = ref.RefGraph.rmat(10, 8, 12)
    off, col, _ = g10.arrays()
    vec["rmat10_off"], vec["rmat10_col"] = off, col
    vec["rmat10_bc1"] = g10.seq_bc(1)
    # RMAT(10,8,21): PR pin graph (test_primitives.cpp:325-340), eps 1e-4
    g21 = ref.RefGraph.rmat(10, 8, 21)
    off, col, _ = g21.arrays()
    vec["rmat10s21_off"], vec["rmat10s21_col"] = off, col
    ranks, it, sums = g21.seq_pagerank(0.85, 1e-4, 1000)
    vec["rmat10s21_pr"], vec["rmat10s21_pr_iters"], vec["rmat10s21_pr_sums"] = ranks, it, sums
    # engine runs: BFS on RMAT(12,16,1) n=4 random(29) with stats
    owner = ref.partition_random(4096, 4, 29)
    plan = ref.RefPlan(g, owner, 4)
    r = plan.bfs(0)
    vec["rmat12_n4_owner"] = owner
    vec["rmat12_n4_bfs_labels"] = r.labels
    vec["rmat12_n4_bfs_S"] = r.stats.supersteps
    vec["rmat12_n4_bfs_W"] = r.stats.edges_examined
    vec["rmat12_n4_bfs_C"] = r.stats.combine_ops
    vec["rmat12_n4_bfs_H"] = r.h_matrix
    r = plan.dobfs(0)
    vec["rmat12_n4_dobfs_dirlog"] = r.direction_log
    vec["rmat12_n4_dobfs_W"] = r.stats.edges_examined
    vec["rmat12_n4_dobfs_H"] = r.h_matrix
    # RMAT-18/16 seed 1 (config 1): BFS labels from source 0 + graph digest
    g18 = ref.RefGraph.rmat(18, 16, 1)
    off18, col18, _ = g18.arrays()
    vec["rmat18_nv_ne"] = np.array([len(off18) - 1, len(col18)], np.uint64)
    vec["rmat18_off_digest"] = np.array([int(off18.astype(np.uint64).sum()),
                                         int((col18.astype(np.uint64) * 2654435761 % (1 << 61)).sum())],
                                        np.uint64)
    vec["rmat18_bfs0"] = g18.seq_bfs(0)
    np.savez_compressed(os.path.join(HERE, "ref_vectors.npz"), **vec)
    print("wrote", sorted(vec))


if __name__ == "__main__":
    main()
