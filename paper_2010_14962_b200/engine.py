"""Python mirror of the reference's hot-path API over the C-ABI engine.

The reference's operator surface for this path is the C++ library's
``sum_range`` / ``run_serial`` / ``run_pool`` over a ``JobSpec``
(proj/core/include/qcut/executor.hpp:30-85) and the lossless ``Payload``
(proj/core/include/qcut/serialize.hpp:32-45). ``Engine`` is built from that
payload and answers the same queries on one B200; errors map onto the
reference's exception classes:

    std::invalid_argument -> ValueError
    qcut::RankGuardError  -> RankGuardError (rank, max_rank)
    std::runtime_error    -> RuntimeError

There is no CPU fallback: compute calls need the in-tree CUDA library
(``paper_2010_14962_b200/_lib/libqcut_gpu.so``) and a GPU and fail loudly
otherwise.
"""
from __future__ import annotations

import ctypes
import gzip
import os
import re
from typing import Optional, Union

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libqcut_gpu.so")

QC_OK, QC_EINVAL, QC_ERANK, QC_EINTERNAL = 0, 1, 2, 3
MODES = {"density": 0, "ket": 1}


class RankGuardError(RuntimeError):
    """qcut::RankGuardError (proj/core/include/qcut/contraction.hpp:34-44)."""

    def __init__(self, msg: str):
        super().__init__(msg)
        m = re.search(r"rank-(\d+) tensor.*max rank (\d+)", msg)
        self.rank = int(m.group(1)) if m else -1
        self.max_rank = int(m.group(2)) if m else -1


class PlanStats(ctypes.Structure):
    _fields_ = [
        ("mode", ctypes.c_int32), ("n_cut", ctypes.c_int32), ("n_steps", ctypes.c_int32),
        ("peak_rank", ctypes.c_int32), ("max_rank", ctypes.c_int32), ("batch_bits", ctypes.c_int32),
        ("jobs", ctypes.c_uint64), ("ket_jobs", ctypes.c_uint64), ("chunks", ctypes.c_uint64),
        ("arena_bytes", ctypes.c_uint64), ("n_kernels", ctypes.c_int32),
        ("n_invariant_steps", ctypes.c_int32), ("essential_bytes", ctypes.c_double),
        ("moved_bytes", ctypes.c_double), ("flops", ctypes.c_double),
        ("dominant_kernel", ctypes.c_int32), ("pad0", ctypes.c_int32), ("dominant_bytes", ctypes.c_double),
        ("algo_flops", ctypes.c_double), ("n_amplitudes", ctypes.c_int32), ("amp_bits", ctypes.c_int32),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


# Every symbol include/qcut_gpu.h declares (checked by tests/test_capi.py).
EXPORTS = (
    "qc_engine_create", "qc_engine_create_ex", "qc_engine_create_batch", "qc_engine_destroy", "qc_engine_plan_stats", "qc_engine_step_shapes",
    "qc_engine_sum_range", "qc_engine_slice_values", "qc_engine_ket_sum", "qc_engine_ket_values",
    "qc_engine_ket_sum_batch", "qc_engine_ket_values_batch",
    "qc_engine_last_run", "qc_engine_bench", "qc_engine_describe", "qc_engine_profile_pass", "qc_last_error",
    "qc_version", "qc_contract_pair", "qc_contract_pair_bench", "qc_engine_bench_cold",
)

_lib = None


def load_library() -> ctypes.CDLL:
    """Load the in-tree engine library; raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("QCUT_GPU_LIB", LIB_PATH)  # build-variant experiments (tools/)
    if not os.path.exists(path):
        raise RuntimeError(f"CUDA engine library missing: {path} (run __graft_entry__.build())")
    lib = ctypes.CDLL(path)
    vp, u64, i32, dp = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.POINTER(ctypes.c_double)
    pi = ctypes.POINTER(ctypes.c_int32)
    lib.qc_engine_create.argtypes = [ctypes.c_char_p, ctypes.c_size_t, i32, i32, u64, ctypes.POINTER(vp)]
    lib.qc_engine_create_ex.argtypes = [ctypes.c_char_p, ctypes.c_size_t, i32, i32, u64, i32, ctypes.POINTER(vp)]
    lib.qc_engine_create_batch.argtypes = [ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_size_t), i32, i32,
                                           i32, u64, i32, ctypes.POINTER(vp)]
    lib.qc_engine_destroy.argtypes = [vp]
    lib.qc_engine_plan_stats.argtypes = [vp, ctypes.POINTER(PlanStats)]
    lib.qc_engine_step_shapes.argtypes = [vp, pi, pi, pi, pi, ctypes.c_size_t]
    for name in ("qc_engine_sum_range", "qc_engine_slice_values", "qc_engine_ket_sum", "qc_engine_ket_values",
                 "qc_engine_ket_sum_batch", "qc_engine_ket_values_batch"):
        getattr(lib, name).argtypes = [vp, u64, u64, dp]
    lib.qc_engine_last_run.argtypes = [vp, dp, ctypes.POINTER(u64), ctypes.POINTER(u64), ctypes.POINTER(u64)]
    lib.qc_engine_bench.argtypes = [vp, i32, u64, u64, dp, dp, dp, dp]
    lib.qc_engine_bench_cold.argtypes = [vp, i32, u64, u64, u64, dp, dp]
    lib.qc_engine_describe.argtypes = [vp, ctypes.c_char_p, ctypes.c_size_t]
    lib.qc_engine_profile_pass.argtypes = [vp, u64, u64, i32, dp, dp, dp, dp, pi, pi]
    lib.qc_contract_pair.argtypes = [i32, i32, i32, dp, pi, i32, dp, pi, i32, i32, i32, dp]
    lib.qc_contract_pair_bench.argtypes = [i32, i32, i32, dp, pi, i32, dp, pi, i32, i32, i32, i32, i32, dp, dp, dp, pi]
    lib.qc_last_error.restype = ctypes.c_char_p
    lib.qc_version.restype = ctypes.c_char_p
    for name in EXPORTS:
        if name not in ("qc_last_error", "qc_version"):
            getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def _raise(rc: int) -> None:
    if rc == QC_OK:
        return
    msg = load_library().qc_last_error().decode()
    if rc == QC_EINVAL:
        raise ValueError(msg)
    if rc == QC_ERANK:
        raise RankGuardError(msg)
    raise RuntimeError(msg)


def _payload_bytes(payload: Union[str, bytes, os.PathLike]) -> bytes:
    if isinstance(payload, bytes):
        return payload
    path = os.fspath(payload)
    if path.lstrip().startswith("{"):
        return path.encode()
    opener = gzip.open if path.endswith(".gz") else open
    with opener(path, "rb") as f:
        return f.read()


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class Engine:
    """One sliced-contraction engine on one device (``device=-1``: host planning only).

    ``mode='density'`` reproduces the reference's own dim-4 view and slice ids;
    ``mode='ket'`` runs the binary-variable view and answers
    density-id queries from the ket slice values.
    """

    def __init__(self, payload, device: int = 0, mode: str = "ket", mem_budget_bytes: int = 0,
                 max_batch_bits: int = -1):
        """``payload``: one payload, or a list of payloads of one network, cut and plan whose
        tensor values differ (output bitstrings, angle sets) -- an amplitude batch: every pass
        computes all of them (``ket_sum_batch`` / ``ket_values_batch``)."""
        if mode not in MODES:
            raise ValueError(f"unknown mode {mode!r}")
        lib = load_library()
        items = list(payload) if isinstance(payload, (list, tuple)) else [payload]
        datas = [_payload_bytes(p) for p in items]
        h = ctypes.c_void_p()
        if len(datas) == 1:
            _raise(lib.qc_engine_create_ex(datas[0], len(datas[0]), device, MODES[mode], mem_budget_bytes,
                                           max_batch_bits, ctypes.byref(h)))
        else:
            arr = (ctypes.c_char_p * len(datas))(*datas)
            lens = (ctypes.c_size_t * len(datas))(*[len(d) for d in datas])
            _raise(lib.qc_engine_create_batch(arr, lens, len(datas), device, MODES[mode], mem_budget_bytes,
                                              max_batch_bits, ctypes.byref(h)))
        self._h = h
        self.mode = mode
        self.device = device
        st = self.plan_stats()
        self.M = st["n_cut"]
        self.n_amplitudes = st["n_amplitudes"]

    def close(self) -> None:
        if getattr(self, "_h", None):
            load_library().qc_engine_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ---- reference API mirror (executor.hpp) ----
    def jobs(self) -> int:
        """JobSpec::jobs() = 4^|cut| (executor.cpp:29-31)."""
        return 4 ** self.M

    def sum_range(self, lo: int, hi: int) -> complex:
        """sum_range(job, lo, hi) (executor.cpp:45-68) over density slice ids."""
        out = np.zeros(2)
        _raise(load_library().qc_engine_sum_range(self._h, lo, hi, _dptr(out)))
        return complex(out[0], out[1])

    def run_serial(self) -> complex:
        """run_serial(job) (executor.cpp:70): the whole range."""
        return self.sum_range(0, self.jobs())

    def slice_values(self, lo: int, hi: int) -> np.ndarray:
        """[sum_range(s, s+1) for s in range(lo, hi)]."""
        out = np.zeros(2 * max(0, hi - lo))
        _raise(load_library().qc_engine_slice_values(self._h, lo, hi, _dptr(out)))
        return out[0::2] + 1j * out[1::2]

    # ---- ket view ----
    def ket_jobs(self) -> int:
        return 2 ** self.M

    def ket_sum(self, klo: int = 0, khi: Optional[int] = None) -> complex:
        """sum of A(k) over ket slice ids [klo, khi) (the amplitude <z|U|0> up to a global phase)."""
        khi = self.ket_jobs() if khi is None else khi
        out = np.zeros(2)
        _raise(load_library().qc_engine_ket_sum(self._h, klo, khi, _dptr(out)))
        return complex(out[0], out[1])

    def ket_values(self, klo: int = 0, khi: Optional[int] = None) -> np.ndarray:
        khi = self.ket_jobs() if khi is None else khi
        out = np.zeros(2 * max(0, khi - klo))
        _raise(load_library().qc_engine_ket_values(self._h, klo, khi, _dptr(out)))
        return out[0::2] + 1j * out[1::2]

    def ket_sum_batch(self, klo: int = 0, khi: Optional[int] = None) -> np.ndarray:
        """Every batched amplitude's sum of A(k) over ket ids [klo, khi) (complex array, one per payload)."""
        khi = self.ket_jobs() if khi is None else khi
        out = np.zeros(2 * self.n_amplitudes)
        _raise(load_library().qc_engine_ket_sum_batch(self._h, klo, khi, _dptr(out)))
        return out[0::2] + 1j * out[1::2]

    def ket_values_batch(self, klo: int = 0, khi: Optional[int] = None) -> np.ndarray:
        """(n_amplitudes, khi - klo) array of A_a(k)."""
        khi = self.ket_jobs() if khi is None else khi
        out = np.zeros(2 * self.n_amplitudes * max(0, khi - klo))
        _raise(load_library().qc_engine_ket_values_batch(self._h, klo, khi, _dptr(out)))
        return (out[0::2] + 1j * out[1::2]).reshape(self.n_amplitudes, max(0, khi - klo))

    # ---- introspection ----
    def plan_stats(self) -> dict:
        st = PlanStats()
        _raise(load_library().qc_engine_plan_stats(self._h, ctypes.byref(st)))
        return st.as_dict()

    def step_shapes(self) -> np.ndarray:
        """(n_steps, 4) array of (rank_a, rank_b, shared legs, result_rank)."""
        n = self.plan_stats()["n_steps"]
        cols = [np.zeros(n, dtype=np.int32) for _ in range(4)]
        ptrs = [c.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)) for c in cols]
        _raise(load_library().qc_engine_step_shapes(self._h, *ptrs, n))
        return np.stack(cols, axis=1)

    def profile_pass(self, lo: int = 0, hi: Optional[int] = None) -> list:
        """One instrumented pass: [{'kind','ms','bytes','flops','exec_flops'}] per launch (CUDA
        events); exec_flops = the flops left after the zero-skip (fused pair kernels)."""
        hi = (2 ** (self.M if self.mode == "ket" else 2 * self.M)) if hi is None else hi
        cap = 4096
        ms, by, fl, ex = np.zeros(cap), np.zeros(cap), np.zeros(cap), np.zeros(cap)
        kd = np.zeros(cap, dtype=np.int32)
        n = ctypes.c_int32()
        _raise(load_library().qc_engine_profile_pass(self._h, lo, hi, cap, _dptr(ms), _dptr(by), _dptr(fl),
                                                     _dptr(ex), kd.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                                     ctypes.byref(n)))
        names = {0: "k_flow", 1: "k_gate", 2: "k_chain", 3: "k_pair", 4: "k_forest", 5: "k_zgemm_dmma"}
        return [{"kind": names.get(int(kd[i]), "?"), "ms": float(ms[i]), "bytes": float(by[i]),
                 "flops": float(fl[i]), "exec_flops": float(ex[i])} for i in range(min(n.value, cap))]

    def describe(self) -> str:
        buf = ctypes.create_string_buffer(1 << 16)
        _raise(load_library().qc_engine_describe(self._h, buf, len(buf)))
        return buf.value.decode()

    def last_run(self) -> dict:
        ms = ctypes.c_double()
        la, h2d, d2h = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        _raise(load_library().qc_engine_last_run(self._h, ctypes.byref(ms), ctypes.byref(la),
                                                 ctypes.byref(h2d), ctypes.byref(d2h)))
        return {"device_ms": ms.value, "launches": la.value, "h2d_bytes": h2d.value, "d2h_bytes": d2h.value}

    def bench(self, reps: int, lo: int = 0, hi: Optional[int] = None) -> dict:
        """Device-resident passes (no host copies), CUDA-event timed; plus the dominant kernel."""
        hi = (2 ** (self.M if self.mode == "ket" else 2 * self.M)) if hi is None else hi
        pass_ms = np.zeros(max(1, reps))
        dom_ms, dom_bytes = ctypes.c_double(), ctypes.c_double()
        out = np.zeros(2)
        _raise(load_library().qc_engine_bench(self._h, reps, lo, hi, _dptr(pass_ms), ctypes.byref(dom_ms),
                                              ctypes.byref(dom_bytes), _dptr(out)))
        return {"pass_ms": pass_ms[:reps].tolist(), "dominant_ms": dom_ms.value,
                "dominant_bytes": dom_bytes.value, "value": complex(out[0], out[1])}


    def bench_cold(self, reps: int, lo: int = 0, hi: Optional[int] = None, flush_bytes: int = 512 << 20) -> dict:
        """As bench(), every timed call behind a device write of ``flush_bytes`` (cold L2) that
        is enqueued on the engine stream outside the call's CUDA-event bracket."""
        hi = (2 ** (self.M if self.mode == "ket" else 2 * self.M)) if hi is None else hi
        pass_ms = np.zeros(max(1, reps))
        out = np.zeros(2)
        _raise(load_library().qc_engine_bench_cold(self._h, reps, lo, hi, flush_bytes, _dptr(pass_ms), _dptr(out)))
        return {"pass_ms": pass_ms[:reps].tolist(), "value": complex(out[0], out[1])}


K_DEFAULT_MAX_RANK = 13  # qcut::kDefaultMaxRank (proj/core/include/qcut/contraction.hpp:32)
PAIR_PATHS = {"auto": 0, "dmma": 1, "dfma": 2, "small": 3}


def _pair_args(a, legs_a, b, legs_b, dim):
    a = np.ascontiguousarray(a, dtype=np.complex128).ravel()
    b = np.ascontiguousarray(b, dtype=np.complex128).ravel()

    def rank_of(t):
        r = int(round(np.log(t.size) / np.log(dim))) if t.size > 0 else -1
        if r < 0 or dim ** r != t.size:
            raise ValueError(f"tensor of {t.size} elements is not a power of the leg dimension {dim}")
        return r

    ra, rb = rank_of(a), rank_of(b)
    # contraction.cpp:74-81 (the C-ABI carries one shared count, so the length check lives here)
    if len(legs_a) == 0 or len(legs_b) == 0:
        raise ValueError("contract_pair needs at least one shared leg")
    if len(legs_a) != len(legs_b):
        raise ValueError(f"shared leg lists differ in length: {len(legs_a)} vs {len(legs_b)}")
    la = np.asarray(legs_a, dtype=np.int32)
    lb = np.asarray(legs_b, dtype=np.int32)
    return a, ra, la, b, rb, lb


def contract_pair(a, legs_a, b, legs_b, max_rank: int = K_DEFAULT_MAX_RANK, dim: int = 4, device: int = 0,
                  path: str = "auto") -> np.ndarray:
    """qcut::contract_pair (proj/core/src/contraction.cpp:71-116) on the device.

    ``a`` / ``b``: row-major complex128 tensors whose legs all have dimension ``dim``; returns the
    flat result tensor (legs: a's free legs in order, then b's). Raises ValueError /
    RankGuardError exactly where the reference throws. No CPU fallback.
    """
    lib = load_library()
    a, ra, la, b, rb, lb = _pair_args(a, legs_a, b, legs_b, dim)
    out_rank = ra + rb - 2 * len(la)
    out = np.empty(max(dim ** max(out_rank, 0), 1), dtype=np.complex128)
    pi = ctypes.POINTER(ctypes.c_int32)
    _raise(lib.qc_contract_pair(device, dim, ra, _dptr(a.view(np.float64)), la.ctypes.data_as(pi), rb,
                                _dptr(b.view(np.float64)), lb.ctypes.data_as(pi), len(la), max_rank,
                                PAIR_PATHS[path], _dptr(out.view(np.float64))))
    return out


def contract_pair_bench(a, legs_a, b, legs_b, dim: int = 4, device: int = 0, path: str = "auto", reps: int = 20,
                        warmup: int = 3, flush_l2: bool = False, e2e: bool = True) -> dict:
    """BM_ContractPair (proj/benchmarks/bench_main.cpp:42-65) on the device: mean kernel time
    with resident operands (CUDA events on the launch stream) and the end-to-end time of one
    call with host buffers. Returns the result too (``out``)."""
    lib = load_library()
    a, ra, la, b, rb, lb = _pair_args(a, legs_a, b, legs_b, dim)
    out = np.empty(dim ** (ra + rb - 2 * len(la)), dtype=np.complex128)
    pi = ctypes.POINTER(ctypes.c_int32)
    kms, ems, used = ctypes.c_double(), ctypes.c_double(), ctypes.c_int32()
    _raise(lib.qc_contract_pair_bench(device, dim, ra, _dptr(a.view(np.float64)), la.ctypes.data_as(pi), rb,
                                      _dptr(b.view(np.float64)), lb.ctypes.data_as(pi), len(la),
                                      PAIR_PATHS[path], reps, warmup, int(flush_l2), _dptr(out.view(np.float64)),
                                      ctypes.byref(kms), ctypes.byref(ems) if e2e else None, ctypes.byref(used)))
    names = {v: k for k, v in PAIR_PATHS.items()}
    k = len(la)
    return {"kernel_ms": kms.value, "e2e_ms": ems.value if e2e else None, "path": names[used.value], "out": out,
            "M": dim ** (ra - k), "N": dim ** (rb - k), "K": dim ** k,
            "flops": 8.0 * dim ** (ra + rb - k)}
