"""TEST INFRASTRUCTURE — the CPU checkers for the PagedEviction hot path.

Two checkers live here; neither is ever on the product path (the CUDA
engine in ``paper_2509_04377_b200`` has no CPU fallback and never imports
this package):

* ``Oracle`` / ``OracleEngine`` — ctypes over ``lib/libpe_oracle.so``, the
  plain-C restatement in ``pe_oracle.c`` (each function cites the reference
  file:line it restates).
* ``Reference`` / ``RefSession`` — ctypes over ``_ref/libpagedevict_ref.so``,
  the UNMODIFIED reference core compiled from ``/root/reference`` plus the
  harness ``ref_harness.cpp``. It pins the restatement (tests/
  test_oracle_pinning.py) and is the CPU baseline of ``bench.py``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
reference / cpu_baseline legs may import this package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "lib" / "libpe_oracle.so"
REF_SO = HERE / "_ref" / "libpagedevict_ref.so"
REF_SRC = Path(os.environ.get("PE_REFERENCE_CORE", "/root/reference/proj/core"))

F32, BF16 = 0, 1
PAGED_EVICTION, FULL_CACHE = 0, 4


def build(force: bool = False) -> None:
    """Build the C restatement (always possible) and, when the reference
    sources are present, the reference library."""
    targets = ["oracle"]
    if REF_SRC.exists():
        targets.append("ref")
    cmd = ["make", "-s", "-C", str(HERE)] + (["-B"] if force else []) + targets
    subprocess.run(cmd, check=True)


def _load(path: Path) -> C.CDLL:
    if not path.exists():
        build()
    if not path.exists():
        raise FileNotFoundError(f"{path} is not built (reference sources absent?)")
    return C.CDLL(str(path))


_p = np.ctypeslib.ndpointer
_dp = C.POINTER(C.c_double)


def _ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


def dtype_code(a: np.ndarray) -> int:
    if a.dtype == np.float32:
        return F32
    if a.dtype == np.uint16:  # bf16 bit patterns
        return BF16
    raise TypeError(f"unsupported element type {a.dtype}")


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bf16 bit patterns (NaN-free inputs)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounding = ((u >> 16) & 1) + 0x7FFF
    return ((u + rounding) >> 16).astype(np.uint16)


class Oracle:
    """Free functions of the C restatement."""

    def __init__(self) -> None:
        lib = _load(ORACLE_SO)
        lib.peo_l2_norm.restype = C.c_double
        lib.peo_l2_norm.argtypes = [C.c_void_p, C.c_size_t, C.c_int]
        lib.peo_token_score.restype = C.c_double
        lib.peo_token_score.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
        lib.peo_rank_tokens.restype = C.c_int
        lib.peo_rank_tokens.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t, C.c_void_p]
        lib.peo_rank_pages.restype = C.c_int64
        lib.peo_rank_pages.argtypes = [C.c_void_p, C.c_size_t]
        lib.peo_output_deviation.restype = C.c_double
        lib.peo_output_deviation.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
        lib.peo_attend_dense.restype = None
        lib.peo_attend_dense.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                                         C.c_size_t, C.c_void_p]
        self.lib = lib

    def l2_norm(self, x: np.ndarray) -> float:
        x = np.ascontiguousarray(x)
        return self.lib.peo_l2_norm(_ptr(x), x.size, dtype_code(x))

    def token_score(self, k: np.ndarray, v: np.ndarray) -> float:
        k = np.ascontiguousarray(k)
        v = np.ascontiguousarray(v)
        return self.lib.peo_token_score(_ptr(k), _ptr(v), k.size, dtype_code(k))

    def rank_tokens(self, positions, scores, k: int) -> np.ndarray:
        pos = np.ascontiguousarray(positions, dtype=np.int64)
        sc = np.ascontiguousarray(scores, dtype=np.float64)
        out = np.zeros(max(k, 1), dtype=np.int64)
        st = self.lib.peo_rank_tokens(_ptr(pos), _ptr(sc), pos.size, k, _ptr(out))
        if st != 0:
            raise KTooLarge(f"k = {k} exceeds {pos.size} scored tokens")
        return out[:k]

    def rank_pages(self, scores) -> int:
        sc = np.ascontiguousarray(scores, dtype=np.float64)
        r = self.lib.peo_rank_pages(_ptr(sc), sc.size)
        if r < 0:
            raise NoEligiblePage("no eligible page to rank")
        return int(r)

    def output_deviation(self, a, b) -> float:
        a = np.ascontiguousarray(a, dtype=np.float32)
        b = np.ascontiguousarray(b, dtype=np.float32)
        if a.size != b.size:
            raise LengthMismatch("deviation requires equal-length vectors")
        return self.lib.peo_output_deviation(_ptr(a), _ptr(b), a.size)

    def attend_dense(self, q, keys, values) -> np.ndarray:
        q = np.ascontiguousarray(q, dtype=np.float32)
        keys = np.ascontiguousarray(keys, dtype=np.float32)
        values = np.ascontiguousarray(values, dtype=np.float32)
        out = np.zeros(q.size, dtype=np.float32)
        self.lib.peo_attend_dense(_ptr(q), _ptr(keys), _ptr(values), keys.shape[0], q.size,
                                  _ptr(out))
        return out


class OracleError(RuntimeError):
    pass


class KTooLarge(OracleError):
    pass


class NoEligiblePage(OracleError):
    pass


class LengthMismatch(OracleError):
    pass


class _PeoEngine(C.Structure):
    _fields_ = [
        ("n_seqs", C.c_int32), ("n_layers", C.c_int32), ("n_tab_heads", C.c_int32),
        ("width", C.c_int32), ("page_size", C.c_int32), ("budget", C.c_int32),
        ("dtype", C.c_int32), ("policy", C.c_int32), ("capacity", C.c_int32),
        ("max_pages", C.c_int32), ("n_tables", C.c_int32),
        ("pages", C.c_void_p), ("positions", C.c_void_p), ("token_scores", C.c_void_p),
        ("page_scores", C.c_void_p), ("block_table", C.c_void_p), ("num_pages", C.c_void_p),
        ("newest_fill", C.c_void_p), ("retained", C.c_void_p), ("stack", C.c_void_p),
        ("top", C.c_int32), ("status", C.c_int32),
    ]


class OracleEngine:
    """The C restatement of the batched engine semantics (same HBM layout as
    the CUDA engine: pages [cap][2][B][w], positions [cap][B], block_table
    [tables][max_pages], LIFO free stack)."""

    def __init__(self, *, n_seqs, n_layers, n_tab_heads, width, page_size, budget, dtype,
                 capacity, max_pages, policy=PAGED_EVICTION):
        self.lib = lib = _load(ORACLE_SO)
        lib.peo_engine_create.restype = C.c_int
        lib.peo_engine_create.argtypes = [C.POINTER(C.POINTER(_PeoEngine))] + [C.c_int32] * 10
        lib.peo_engine_destroy.argtypes = [C.POINTER(_PeoEngine)]
        lib.peo_prefill.argtypes = [C.POINTER(_PeoEngine), C.c_int32, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]
        lib.peo_decode_append.argtypes = [C.POINTER(_PeoEngine), C.c_int32, C.c_int32,
                                          C.c_void_p, C.c_void_p, C.c_void_p]
        lib.peo_decode_evict.argtypes = [C.POINTER(_PeoEngine), C.c_int32, C.c_int32, C.c_void_p]
        lib.peo_attention.argtypes = [C.POINTER(_PeoEngine), C.c_int32, C.c_void_p, C.c_int32,
                                      C.c_void_p]
        self.dtype = dtype
        h = C.POINTER(_PeoEngine)()
        st = lib.peo_engine_create(C.byref(h), n_seqs, n_layers, n_tab_heads, width, page_size,
                                   budget, dtype, policy, capacity, max_pages)
        if st != 0:
            raise OracleError(f"peo_engine_create failed with status {st}")
        self.h = h
        self.e = h.contents
        self.n_tab_heads = n_tab_heads
        self.n_seqs = n_seqs
        self.n_layers = n_layers

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.peo_engine_destroy(self.h)
            self.h = None

    def _arr(self, ptr, n, dt):
        buf = (C.c_char * (n * np.dtype(dt).itemsize)).from_address(ptr)
        return np.frombuffer(buf, dtype=dt, count=n)

    # state views (copies)
    @property
    def top(self) -> int:
        return self.e.top

    def block_table(self) -> np.ndarray:
        e = self.e
        return self._arr(e.block_table, e.n_tables * e.max_pages, np.int32).reshape(
            e.n_tables, e.max_pages).copy()

    def num_pages(self):
        return self._arr(self.e.num_pages, self.e.n_tables, np.int32).copy()

    def newest_fill(self):
        return self._arr(self.e.newest_fill, self.e.n_tables, np.int32).copy()

    def retained(self):
        return self._arr(self.e.retained, self.e.n_tables, np.int32).copy()

    def free_stack(self):
        return self._arr(self.e.stack, self.e.capacity, np.int32)[: self.e.top].copy()

    def positions(self):
        e = self.e
        return self._arr(e.positions, e.capacity * e.page_size, np.int32).reshape(
            e.capacity, e.page_size).copy()

    def page_scores(self):
        return self._arr(self.e.page_scores, self.e.capacity, np.float64).copy()

    def token_scores(self):
        e = self.e
        return self._arr(e.token_scores, e.capacity * e.page_size, np.float64).reshape(
            e.capacity, e.page_size).copy()

    def pages(self):
        e = self.e
        dt = np.uint16 if e.dtype == BF16 else np.float32
        return self._arr(e.pages, e.capacity * 2 * e.page_size * e.width, dt).reshape(
            e.capacity, 2, e.page_size, e.width).copy()

    # operations
    def prefill(self, layer, k, v, cu_seqlens, seq_begin=0):
        cu = np.ascontiguousarray(cu_seqlens, dtype=np.int32)
        n = cu.size - 1
        ev = np.zeros(max(n * self.n_tab_heads, 1), dtype=np.int32)
        k = np.ascontiguousarray(k)
        v = np.ascontiguousarray(v)
        st = self.lib.peo_prefill(self.h, layer, _ptr(k), _ptr(v), _ptr(cu), seq_begin, n,
                                  _ptr(ev))
        return st, ev[: n * self.n_tab_heads]

    def decode_append(self, layer_begin, n_layers, k, v, positions):
        k = np.ascontiguousarray(k)
        v = np.ascontiguousarray(v)
        pos = np.ascontiguousarray(positions, dtype=np.int64)
        return self.lib.peo_decode_append(self.h, layer_begin, n_layers, _ptr(k), _ptr(v),
                                          _ptr(pos))

    def decode_evict(self, layer_begin, n_layers):
        n = n_layers * self.n_seqs * self.n_tab_heads
        vic = np.zeros(n, dtype=np.int32)
        st = self.lib.peo_decode_evict(self.h, layer_begin, n_layers, _ptr(vic))
        return st, vic

    def attention(self, layer, q, G):
        q = np.ascontiguousarray(q)
        out = np.zeros(q.shape, dtype=np.float32)
        st = self.lib.peo_attention(self.h, layer, _ptr(q), G, _ptr(out))
        return st, out

    def table_id(self, seq, layer, head):
        return (seq * self.n_layers + layer) * self.n_tab_heads + head


class Reference:
    """ctypes over the compiled reference library + harness."""

    def __init__(self) -> None:
        lib = _load(REF_SO)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_l2_norm.restype = C.c_double
        lib.ref_l2_norm.argtypes = [C.c_void_p, C.c_size_t]
        lib.ref_token_importance.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, _dp]
        lib.ref_rank_tokens.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t, C.c_void_p]
        lib.ref_rank_pages.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]
        lib.ref_validate_config.argtypes = [C.c_size_t, C.c_uint32, C.c_size_t, C.c_int]
        lib.ref_memory_bytes.argtypes = [C.c_uint64] * 5 + [C.POINTER(C.c_uint64)]
        lib.ref_attend_dense.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p,
                                         C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p]
        lib.ref_output_deviation.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, _dp]
        lib.ref_session_create.restype = C.c_void_p
        lib.ref_session_create.argtypes = [C.c_size_t, C.c_uint32, C.c_size_t, C.c_int, C.c_size_t,
                                           C.c_uint32, C.POINTER(C.c_int)]
        lib.ref_session_destroy.argtypes = [C.c_void_p]
        lib.ref_prefill.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p, C.c_size_t,
                                    C.c_void_p, C.c_void_p, C.POINTER(C.c_size_t)]
        lib.ref_decode_step.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p,
                                        C.c_uint64, C.c_int64, C.POINTER(C.c_int),
                                        C.POINTER(C.c_int64)]
        lib.ref_page_count.restype = C.c_size_t
        lib.ref_page_count.argtypes = [C.c_void_p, C.c_size_t]
        lib.ref_retained_len.restype = C.c_size_t
        lib.ref_retained_len.argtypes = [C.c_void_p, C.c_size_t]
        lib.ref_fragmentation.restype = None
        lib.ref_fragmentation.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p]
        lib.ref_append_token.restype = C.c_int
        lib.ref_append_token.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p, C.c_uint64]
        lib.ref_policy_evict.restype = C.c_int
        lib.ref_policy_evict.argtypes = [C.c_void_p, C.c_size_t, C.c_uint64, C.c_int64,
                                         C.POINTER(C.c_int), C.POINTER(C.c_int64)]
        lib.ref_free_count.restype = C.c_size_t
        lib.ref_free_count.argtypes = [C.c_void_p]
        lib.ref_read_table.argtypes = [C.c_void_p, C.c_size_t] + [C.c_void_p] * 5
        lib.ref_mirror_free_list.restype = C.c_size_t
        lib.ref_mirror_free_list.argtypes = [C.c_void_p, C.c_void_p]
        lib.ref_drain_free_list.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_size_t), C.c_int]
        lib.ref_attend_table.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_uint32,
                                         C.c_uint32, C.c_void_p]
        lib.ref_bench_decode_cycles.argtypes = [C.c_size_t, C.c_size_t, C.c_uint32, C.c_uint32,
                                                C.c_size_t, C.c_size_t, C.c_size_t, C.c_uint64, _dp,
                                                C.POINTER(C.c_uint64)]
        lib.ref_bench_prefill.argtypes = [C.c_size_t, C.c_size_t, C.c_size_t, C.c_uint32,
                                          C.c_uint32, C.c_size_t, C.c_uint64, _dp]
        lib.ref_bench_attend.argtypes = [C.c_size_t, C.c_size_t, C.c_uint32, C.c_uint32,
                                         C.c_uint32, C.c_size_t, C.c_uint64, _dp]
        self.lib = lib

    def _check(self, st: int) -> None:
        if st != 0:
            raise RefError(st, self.lib.ref_last_error().decode())

    def l2_norm(self, x) -> float:
        x = np.ascontiguousarray(x, dtype=np.float32)
        return self.lib.ref_l2_norm(_ptr(x), x.size)

    def token_importance(self, k, v) -> float:
        k = np.ascontiguousarray(k, dtype=np.float32)
        v = np.ascontiguousarray(v, dtype=np.float32)
        out = C.c_double()
        self._check(self.lib.ref_token_importance(_ptr(k), _ptr(v), k.size, C.byref(out)))
        return out.value

    def rank_tokens(self, positions, scores, k) -> np.ndarray:
        pos = np.ascontiguousarray(positions, dtype=np.uint64)
        sc = np.ascontiguousarray(scores, dtype=np.float64)
        out = np.zeros(max(k, 1), dtype=np.uint64)
        self._check(self.lib.ref_rank_tokens(_ptr(pos), _ptr(sc), pos.size, k, _ptr(out)))
        return out[:k].astype(np.int64)

    def rank_pages(self, scores) -> int:
        sc = np.ascontiguousarray(scores, dtype=np.float64)
        out = C.c_size_t()
        self._check(self.lib.ref_rank_pages(_ptr(sc), sc.size, C.byref(out)))
        return out.value

    def validate_config(self, budget, page_size, sinks=4, kind=PAGED_EVICTION) -> int:
        return self.lib.ref_validate_config(budget, page_size, sinks, kind)

    def memory_bytes(self, *args) -> int:
        out = C.c_uint64()
        self._check(self.lib.ref_memory_bytes(*args, C.byref(out)))
        return out.value

    def attend_dense(self, keys, values, query, heads, dim, page_size=16) -> np.ndarray:
        keys = np.ascontiguousarray(keys, dtype=np.float32)
        values = np.ascontiguousarray(values, dtype=np.float32)
        query = np.ascontiguousarray(query, dtype=np.float32)
        out = np.zeros(heads * dim, dtype=np.float32)
        self._check(self.lib.ref_attend_dense(_ptr(keys), _ptr(values), keys.shape[0],
                                              _ptr(query), heads, dim, page_size, _ptr(out)))
        return out

    def output_deviation(self, a, b) -> float:
        a = np.ascontiguousarray(a, dtype=np.float32)
        b = np.ascontiguousarray(b, dtype=np.float32)
        out = C.c_double()
        self._check(self.lib.ref_output_deviation(_ptr(a), a.size, _ptr(b), b.size, C.byref(out)))
        return out.value

    def session(self, capacity, page_size, budget, n_tables, width, kind=PAGED_EVICTION):
        return RefSession(self, capacity, page_size, budget, n_tables, width, kind)

    def bench_decode_cycles(self, n_tables, budget, page_size, w, threads, cycles, seed=1,
                            warmup_cycles=0):
        """Times `cycles` eviction cycles (after `warmup_cycles` untimed ones)
        of the reference's decode_step on `n_tables` tables; returns
        (seconds, page evictions in the timed cycles)."""
        secs = C.c_double()
        ev = C.c_uint64()
        self._check(self.lib.ref_bench_decode_cycles(n_tables, budget, page_size, w, threads,
                                                     warmup_cycles, cycles, seed, C.byref(secs),
                                                     C.byref(ev)))
        return secs.value, ev.value

    def bench_prefill(self, n_tables, L, budget, page_size, w, threads, seed=1):
        secs = C.c_double()
        self._check(self.lib.ref_bench_prefill(n_tables, L, budget, page_size, w, threads, seed,
                                               C.byref(secs)))
        return secs.value

    def bench_attend(self, n_tables, R, page_size, d, G, threads, seed=1):
        secs = C.c_double()
        self._check(self.lib.ref_bench_attend(n_tables, R, page_size, d, G, threads, seed,
                                              C.byref(secs)))
        return secs.value


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class RefSession:
    """One reference PagePool + BlockTable/EvictionPolicy per table."""

    def __init__(self, ref: Reference, capacity, page_size, budget, n_tables, width, kind):
        self.ref = ref
        self.lib = ref.lib
        st = C.c_int()
        self.h = self.lib.ref_session_create(capacity, page_size, budget, kind, n_tables, width,
                                             C.byref(st))
        if st.value != 0:
            raise RefError(st.value, self.lib.ref_last_error().decode())
        self.width = width
        self.capacity = capacity

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_session_destroy(self.h)
            self.h = None

    def prefill(self, t, k, v, positions=None):
        k = np.ascontiguousarray(k, dtype=np.float32)
        v = np.ascontiguousarray(v, dtype=np.float32)
        L = k.shape[0]
        pos = np.arange(L, dtype=np.uint64) if positions is None else np.ascontiguousarray(
            positions, dtype=np.uint64)
        ev = np.zeros(max(L, 1), dtype=np.uint64)
        n = C.c_size_t()
        self.ref._check(self.lib.ref_prefill(self.h, t, _ptr(k), _ptr(v), L, _ptr(pos), _ptr(ev),
                                             C.byref(n)))
        return ev[: n.value].astype(np.int64)

    def decode_step(self, t, k, v, position, step):
        k = np.ascontiguousarray(k, dtype=np.float32)
        v = np.ascontiguousarray(v, dtype=np.float32)
        kind = C.c_int()
        idx = C.c_int64()
        self.ref._check(self.lib.ref_decode_step(self.h, t, _ptr(k), _ptr(v), position, step,
                                                 C.byref(kind), C.byref(idx)))
        return kind.value, idx.value

    def page_count(self, t) -> int:
        return self.lib.ref_page_count(self.h, t)

    def retained_len(self, t) -> int:
        return self.lib.ref_retained_len(self.h, t)

    def append_token(self, t, k, v, position) -> None:
        """BlockTable::append_token alone (phase 1 of a two-phase step)."""
        k = np.ascontiguousarray(k, dtype=np.float32)
        v = np.ascontiguousarray(v, dtype=np.float32)
        self.ref._check(self.lib.ref_append_token(self.h, t, _ptr(k), _ptr(v), int(position)))

    def policy_evict(self, t, newest, step) -> tuple[int, int]:
        """The policy's evict after the append: (kind, victim position or
        logical page, -1 if none)."""
        kind, victim = C.c_int(0), C.c_int64(-1)
        self.ref._check(self.lib.ref_policy_evict(self.h, t, int(newest), int(step), C.byref(kind),
                                                  C.byref(victim)))
        return kind.value, victim.value

    def fragmentation(self, t) -> tuple[float, float]:
        """(fragmentation_ratio, fragmentation_ratio_excluding_newest)."""
        out = (C.c_double * 2)()
        self.lib.ref_fragmentation(self.h, t, out)
        return out[0], out[1]

    def free_count(self) -> int:
        return self.lib.ref_free_count(self.h)

    def read_table(self, t, with_data=True):
        n = self.page_count(t)
        r = self.retained_len(t)
        phys = np.zeros(max(n, 1), dtype=np.uint32)
        fills = np.zeros(max(n, 1), dtype=np.uint32)
        pos = np.zeros(max(r, 1), dtype=np.uint64)
        keys = np.zeros((max(r, 1), self.width), dtype=np.float32) if with_data else None
        vals = np.zeros((max(r, 1), self.width), dtype=np.float32) if with_data else None
        self.ref._check(self.lib.ref_read_table(
            self.h, t, _ptr(phys), _ptr(fills), _ptr(pos),
            _ptr(keys) if with_data else None, _ptr(vals) if with_data else None))
        out = dict(phys=phys[:n].astype(np.int64), fills=fills[:n].astype(np.int64),
                   positions=pos[:r].astype(np.int64))
        if with_data:
            out["keys"] = keys[:r]
            out["values"] = vals[:r]
        return out

    def mirror_free_list(self) -> np.ndarray:
        out = np.zeros(max(self.capacity, 1), dtype=np.uint32)
        n = self.lib.ref_mirror_free_list(self.h, _ptr(out))
        return out[:n].astype(np.int64)

    def drain_free_list(self, check_mirror: bool = True) -> np.ndarray:
        """Drains the real pool (allocate() until empty); with check_mirror
        the order must equal the harness's free-list mirror."""
        out = np.zeros(max(self.capacity, 1), dtype=np.uint32)
        n = C.c_size_t()
        self.ref._check(self.lib.ref_drain_free_list(self.h, _ptr(out), C.byref(n), int(check_mirror)))
        return out[: n.value].astype(np.int64)

    def attend(self, t, q, heads, dim):
        q = np.ascontiguousarray(q, dtype=np.float32)
        out = np.zeros(heads * dim, dtype=np.float32)
        self.ref._check(self.lib.ref_attend_table(self.h, t, _ptr(q), heads, dim, _ptr(out)))
        return out
