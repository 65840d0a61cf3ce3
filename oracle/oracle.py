"""CPU oracle — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or the
timed CPU baseline. The product package never imports it.

It wraps ``oracle/_ref/liboracle.so`` (``qcut_oracle.c``, a plain-C restatement of
the reference's sum_range → apply_cut → execute_plan → contract_pair path, see the
file header for the reference file:line of every function) and adds:

* ``load_payload``: parse the reference's ``encode_payload`` JSON
  (proj/core/src/serialize.cpp:147-154, network dump tensor_network.cpp:179-196)
* ``ket_factor``: the ket view of a density-basis tensor (SURVEY.md §8 conventions):
  a reference tensor over dim-4 legs whose digit is a = 2*ket + bra
  (tensor_network.cpp:25-32) factorises as T = K (x) conj(K) for pure inputs,
  unitary gates and projector measurements; K is recovered with a fixed phase
  convention (the largest-magnitude diagonal entry of K real positive).
* ``refgen``: run the compiled reference driver (oracle/_ref/qcut_refgen).

Parity status: pinned — tests/test_oracle_golden.py checks this oracle against
the compiled, unmodified reference's outputs stored in tests/golden/.
"""
from __future__ import annotations

import ctypes
import gzip
import json
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
LIB_PATH = os.path.join(REF_DIR, "liboracle.so")
REFGEN = os.path.join(REF_DIR, "qcut_refgen")


def build(ref: bool = True) -> None:
    """Compile the oracle (and, when /root/reference exists, the reference)."""
    targets = ["oracle"]
    if ref and os.path.isdir("/root/reference/proj/core/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-j8", *targets], cwd=HERE, check=True)


def read_json(path: str) -> dict:
    opener = gzip.open if path.endswith(".gz") else open
    with opener(path, "rt") as f:
        return json.load(f)


@dataclass
class Payload:
    """Flattened reference payload: network, cut, plan, max_rank."""

    vid: np.ndarray
    vrank: np.ndarray
    vdata: list  # per-vertex complex128 arrays (dim-4 basis)
    edges: np.ndarray  # (ne, 5): id, u, leg_u, v, leg_v
    cut: list
    steps: list  # dicts from the plan
    scalars: list
    max_rank: int
    peak_rank: int
    raw: dict = field(repr=False, default=None)

    @property
    def M(self) -> int:
        return len(self.cut)


def load_payload(src) -> Payload:
    p = src if isinstance(src, dict) else read_json(src)
    if p.get("v") != 1:
        raise ValueError("unsupported payload version")
    verts = sorted(p["network"]["vertices"], key=lambda v: v["id"])
    vid = np.array([v["id"] for v in verts], dtype=np.int32)
    vrank = np.array([v["rank"] for v in verts], dtype=np.int32)
    vdata = []
    for v in verts:
        d = np.array(v["data"], dtype=np.float64).reshape(-1, 2)
        vdata.append(d[:, 0] + 1j * d[:, 1])
    edges = np.array(
        [[e["id"], e["endpoints"][0][0], e["endpoints"][0][1], e["endpoints"][1][0], e["endpoints"][1][1]]
         for e in p["network"]["edges"]],
        dtype=np.int32,
    ).reshape(-1, 5)
    plan = p["plan"]
    return Payload(vid, vrank, vdata, edges, list(p["cut"]), plan["steps"], list(plan["scalars"]),
                   int(p["max_rank"]), int(plan["peak_rank"]), p)


def ket_factor(t: np.ndarray, rank: int, tol: float = 1e-12) -> np.ndarray:
    """K with T[(k1 b1)...(kr br)] = K[k1..kr] * conj(K[b1..br]); raises if T is not rank 1."""
    if rank == 0:
        return t.copy()
    # density index bits: leg i -> (ket, bra) = bits (2(r-1-i)+1, 2(r-1-i)); reshape to
    # (2,2)*r with axis order k1,b1,k2,b2,... then move kets first.
    v = t.reshape((2, 2) * rank)
    v = v.transpose(list(range(0, 2 * rank, 2)) + list(range(1, 2 * rank, 2)))
    n = 1 << rank
    V = v.reshape(n, n)
    diag = np.abs(np.diag(V))
    j = int(np.argmax(diag))
    if diag[j] == 0.0:
        return np.zeros(n, dtype=np.complex128)
    K = V[:, j] / np.sqrt(V[j, j].real)
    err = np.max(np.abs(V - np.outer(K, K.conj())))
    if err > tol * max(1.0, np.max(np.abs(V))):
        raise ValueError(f"tensor does not factorise as K (x) conj(K) (err {err:.3g})")
    return K


class _Net(ctypes.Structure):
    _fields_ = [
        ("D", ctypes.c_int), ("nv", ctypes.c_int),
        ("vid", ctypes.c_void_p), ("vrank", ctypes.c_void_p), ("voff", ctypes.c_void_p),
        ("vdata", ctypes.c_void_p),
        ("ne", ctypes.c_int),
        ("e_id", ctypes.c_void_p), ("e_u", ctypes.c_void_p), ("e_lu", ctypes.c_void_p),
        ("e_v", ctypes.c_void_p), ("e_lv", ctypes.c_void_p),
        ("M", ctypes.c_int), ("cut", ctypes.c_void_p),
        ("nsteps", ctypes.c_int),
        ("st_a", ctypes.c_void_p), ("st_b", ctypes.c_void_p), ("st_k", ctypes.c_void_p),
        ("st_off", ctypes.c_void_p), ("st_la", ctypes.c_void_p), ("st_lb", ctypes.c_void_p),
        ("nscal", ctypes.c_int), ("scal", ctypes.c_void_p),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build(ref=False)
        _lib = ctypes.CDLL(LIB_PATH)
        _lib.qo_sum_range.restype = ctypes.c_int
        _lib.qo_sum_range.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                      ctypes.c_void_p, ctypes.c_void_p]
        _lib.qo_sum_range_pool.restype = ctypes.c_int
        _lib.qo_sum_range_pool.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                           ctypes.c_int, ctypes.c_void_p]
        _lib.qo_last_error.restype = ctypes.c_char_p
        _lib.qo_contract_pair.restype = ctypes.c_int
    return _lib


def _i32(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32))


class OracleNet:
    """A payload flattened for the C oracle in one view: 'density' (D=4) or 'ket' (D=2)."""

    def __init__(self, payload: Payload, mode: str = "density"):
        if mode not in ("density", "ket"):
            raise ValueError(mode)
        self.payload = payload
        self.mode = mode
        self.D = 4 if mode == "density" else 2
        datas = payload.vdata if mode == "density" else [
            ket_factor(d, int(r)) for d, r in zip(payload.vdata, payload.vrank)]
        sizes = np.array([len(d) for d in datas], dtype=np.int64)
        self.voff = np.ascontiguousarray(np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64))
        flat = np.concatenate(datas).astype(np.complex128)
        self.vdata = np.ascontiguousarray(np.stack([flat.real, flat.imag], axis=1).reshape(-1))
        self.vid = _i32(payload.vid)
        self.vrank = _i32(payload.vrank)
        e = payload.edges
        self.e = [_i32(e[:, i]) for i in range(5)]
        self.cut = _i32(payload.cut if payload.cut else [0])
        st = payload.steps
        self.st_a = _i32([s["a"] for s in st])
        self.st_b = _i32([s["b"] for s in st])
        self.st_k = _i32([len(s["legs_a"]) for s in st])
        self.st_off = _i32(np.concatenate([[0], np.cumsum([len(s["legs_a"]) for s in st])[:-1]]))
        self.st_la = _i32([l for s in st for l in s["legs_a"]] or [0])
        self.st_lb = _i32([l for s in st for l in s["legs_b"]] or [0])
        self.scal = _i32(payload.scalars or [0])
        ptr = lambda a: a.ctypes.data  # noqa: E731
        self.net = _Net(self.D, len(self.vid), ptr(self.vid), ptr(self.vrank), ptr(self.voff),
                        ptr(self.vdata), len(e), *[ptr(a) for a in self.e], payload.M, ptr(self.cut),
                        len(st), ptr(self.st_a), ptr(self.st_b), ptr(self.st_k), ptr(self.st_off),
                        ptr(self.st_la), ptr(self.st_lb), len(payload.scalars), ptr(self.scal))

    @property
    def jobs(self) -> int:
        return self.D ** self.payload.M

    def sum_range(self, lo: int, hi: int, per_slice: bool = False):
        out = np.zeros(2)
        ps = np.zeros(2 * max(0, hi - lo)) if per_slice else None
        rc = lib().qo_sum_range(ctypes.byref(self.net), lo, hi, out.ctypes.data,
                                ps.ctypes.data if ps is not None else None)
        if rc:
            raise ValueError(lib().qo_last_error().decode())
        v = complex(out[0], out[1])
        if per_slice:
            return v, ps[0::2] + 1j * ps[1::2]
        return v

    def sum_range_pool(self, lo: int, hi: int, workers: int) -> complex:
        out = np.zeros(2)
        rc = lib().qo_sum_range_pool(ctypes.byref(self.net), lo, hi, workers, out.ctypes.data)
        if rc:
            raise ValueError(lib().qo_last_error().decode())
        return complex(out[0], out[1])


def contract_pair(D, e, legs_e, f, legs_f):
    """contract_pair (contraction.cpp:71-116) on flat complex arrays; returns a flat array."""
    e = np.ascontiguousarray(e, dtype=np.complex128)
    f = np.ascontiguousarray(f, dtype=np.complex128)
    re = int(round(np.log(len(e)) / np.log(D)))
    rf = int(round(np.log(len(f)) / np.log(D)))
    k = len(legs_e)
    out = np.zeros(D ** (re + rf - 2 * k), dtype=np.complex128)
    le, lf = _i32(legs_e), _i32(legs_f)
    rc = lib().qo_contract_pair(D, re, e.ctypes.data_as(ctypes.c_void_p), le.ctypes.data_as(ctypes.c_void_p),
                                rf, f.ctypes.data_as(ctypes.c_void_p), lf.ctypes.data_as(ctypes.c_void_p),
                                k, out.ctypes.data_as(ctypes.c_void_p))
    if rc:
        raise ValueError("invalid leg lists")
    return out


def refgen(*args: str) -> dict:
    """Run the compiled reference driver and parse its JSON output."""
    out = subprocess.run([REFGEN, *args], check=True, capture_output=True, text=True).stdout
    return json.loads(out.strip().splitlines()[-1])
