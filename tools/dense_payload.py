"""A dense three-tensor network in the reference's payload format (serialize.cpp:147-154).

Vertices A, B, C with a parallel A-B legs, b B-C legs and c A-C legs (every leg of dimension
4), seeded random complex entries, edge 0 (an A-B leg) cut. The plan contracts A with B over
their a - 1 uncut legs -- an M x K x N = 4^c x 4^(a-1) x 4^b dense contraction per slice, the
contract_pair shape BM_ContractPair measures (bench_main.cpp:42-65) -- then the result with C
over all b + c legs. It is the engine's test case for a dense PlanStep (the FP64 tensor-pipe
GEMM inside a pass): QAOA elimination plans have none (every step has one small operand).
tools/make_golden.py --dense runs the UNMODIFIED reference on this payload and records its
values; the payload itself is rebuilt from the seed wherever it is needed.
"""
import json

import numpy as np


def dense_triangle(a=4, b=3, c=3, seed=7, cut=True):
    rng = np.random.default_rng(seed)

    def tensor(rank):
        n = 4 ** rank
        # entries of order 4^(-rank/4): the contracted value stays of order one
        v = (rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)) * 2.0 ** (-rank / 2)
        return v

    ranks = [a + c, a + b, b + c]
    data = [tensor(r) for r in ranks]
    edges = []
    for i in range(a):  # A-B
        edges.append({"id": len(edges), "endpoints": [[0, i], [1, i]]})
    for i in range(b):  # B-C
        edges.append({"id": len(edges), "endpoints": [[1, a + i], [2, i]]})
    for i in range(c):  # A-C
        edges.append({"id": len(edges), "endpoints": [[0, a + i], [2, b + i]]})
    ncut = 1 if cut else 0
    k1 = a - ncut
    step1 = {"a": 0, "b": 1, "out": 0, "edges": list(range(ncut, a)), "legs_a": list(range(k1)),
             "legs_b": list(range(k1)), "rank_a": k1 + c, "rank_b": k1 + b, "result_rank": b + c,
             "work_rank": k1 + b + c}
    # result legs of step 1: A's free legs (A-C edges) then B's free legs (B-C edges)
    step2 = {"a": 0, "b": 2, "out": 0, "edges": list(range(a + b, a + b + c)) + list(range(a, a + b)),
             "legs_a": list(range(b + c)), "legs_b": list(range(b, b + c)) + list(range(b)),
             "rank_a": b + c, "rank_b": b + c, "result_rank": 0, "work_rank": b + c}
    payload = {
        "v": 1, "cut": [0] if cut else [], "max_rank": 13,
        "network": {"v": 1, "edges": edges,
                    "vertices": [{"id": i, "rank": ranks[i], "data": [[float(z.real), float(z.imag)] for z in data[i]]}
                                 for i in range(3)]},
        "plan": {"steps": [step1, step2], "scalars": [], "peak_rank": max(k1 + c, k1 + b, b + c),
                 "cost_estimate": float(4 ** (k1 + b + c) + 4 ** (b + c))},
    }
    return payload, data


def dense_value(a, b, c, data):
    """The closed network's value by numpy (all legs summed): the reference's run_serial."""
    A = data[0].reshape(4 ** a, 4 ** c)
    B = data[1].reshape(4 ** a, 4 ** b)
    C = data[2].reshape(4 ** b, 4 ** c)
    return complex(np.einsum("ac,ab,bc->", A, B, C))


if __name__ == "__main__":
    import sys
    p, d = dense_triangle()
    json.dump(p, open(sys.argv[1], "w"), separators=(",", ":"))
    print(dense_value(4, 3, 3, d))
