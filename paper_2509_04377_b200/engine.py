"""Python mirror of the reference cache-manager API over the B200 engine.

Reference (proj/core/include/pagedevict/): PolicyKind / PolicyConfig
(policy.hpp:17-39), EvictionDecision (policy.hpp:43-84), the Error hierarchy
(errors.hpp:12-88), PagePool (page_pool.hpp:19-42), BlockTable
(block_table.hpp:21-102) and EvictionPolicy::prefill_compress / decode_step
(policy.hpp:95-120). The reference objects are per (sequence, layer) and
mutated one token at a time; here ONE engine owns every table of a rank in
HBM and each call is a batched, stream-ordered launch over many tables
(include/pe.h). Per-table accessors read the device state back.

Buffers may be torch tensors (CUDA or CPU) or numpy arrays; host buffers are
staged by the C-ABI itself.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass

import numpy as np

from . import _lib


# ----------------------------------------------------------------- errors (errors.hpp:12-88)
class Error(RuntimeError):
    status = 1


class PoolExhausted(Error):
    status = 2


class IndexOutOfRange(Error):
    status = 3


class UnknownPosition(Error):
    status = 4


class Overflow(Error):
    status = 5


class EmptyPage(Error):
    status = 6


class KTooLarge(Error):
    status = 7


class NoEligiblePage(Error):
    status = 8


class BudgetInvalid(Error):
    status = 9


class EmptyCache(Error):
    status = 10


class LengthMismatch(Error):
    status = 11


class EmptyInput(Error):
    status = 12


class IoError(Error):
    status = 13


class InvalidArgument(Error):
    status = 20


class InvalidState(Error):
    status = 21


class CudaError(Error):
    status = 30


class NoDevice(Error):
    status = 31


_BY_STATUS = {cls.status: cls for cls in (
    Error, PoolExhausted, IndexOutOfRange, UnknownPosition, Overflow, EmptyPage, KTooLarge,
    NoEligiblePage, BudgetInvalid, EmptyCache, LengthMismatch, EmptyInput, IoError,
    InvalidArgument, InvalidState, CudaError, NoDevice)}


def _check(status: int) -> None:
    if status != 0:
        lib = _lib.load()
        msg = lib.pe_last_error().decode(errors="replace")
        raise _BY_STATUS.get(status, Error)(f"[{status}] {msg}")


# ----------------------------------------------------------------- policy config (policy.hpp:17-39)
class PolicyKind(enum.IntEnum):
    PagedEviction = 0
    StreamingLlm = 1
    InvKeyL2 = 2
    KeyDiff = 3
    FullCache = 4


_NAMES = {PolicyKind.PagedEviction: "paged-eviction", PolicyKind.StreamingLlm: "streaming-llm",
          PolicyKind.InvKeyL2: "inv-key-l2", PolicyKind.KeyDiff: "key-diff",
          PolicyKind.FullCache: "full"}


def to_string(kind: PolicyKind) -> str:
    """policy.cpp:17-27"""
    return _NAMES[PolicyKind(kind)]


def parse_policy_kind(name: str) -> PolicyKind | None:
    """policy.cpp:29-36"""
    for k, v in _NAMES.items():
        if v == name:
            return k
    return None


@dataclass
class PolicyConfig:
    cache_budget: int = 256  # C, tokens
    page_size: int = 16      # B, tokens per page
    sink_count: int = 4      # StreamingLLM only
    kind: PolicyKind = PolicyKind.PagedEviction

    def validate(self) -> None:
        """policy.cpp:38-52"""
        if self.page_size == 0:
            raise BudgetInvalid("page size must be positive")
        if self.cache_budget < self.page_size:
            raise BudgetInvalid(f"budget must be at least one page ({self.page_size} tokens)")
        if self.cache_budget % self.page_size != 0:
            raise BudgetInvalid("budget must be a multiple of page size")
        if self.kind == PolicyKind.StreamingLlm and self.sink_count >= self.cache_budget:
            raise BudgetInvalid("sink count must be smaller than the budget")


class ScoreMode(enum.IntEnum):
    RECOMPUTE = 0  # K2: rescore resident pages from their K/V bytes
    CACHED = 1     # K2c: page means cached when each page filled


class TokenRule(enum.IntEnum):
    """Victim rules of the unstructured baselines (pe_token_rule, pe.h)."""
    AT_POSITION = 0   # BlockTable::evict_slot
    STREAMING = 1     # StreamingLlmPolicy::evict (arg = sink count)
    MAX_KEY_NORM = 2  # InvKeyL2Policy::evict
    KEY_DIFF = 3      # KeyDiffPolicy::evict


class Granularity(enum.IntEnum):
    PER_KV_HEAD = 0
    PER_LAYER = 1


DTYPE_F32, DTYPE_BF16 = 0, 1


# ----------------------------------------------------------------- buffers
def _ptr(buf):
    """(pointer, keepalive) for a torch tensor / numpy array / None."""
    if buf is None:
        return None, None
    if hasattr(buf, "data_ptr"):
        if not buf.is_contiguous():
            raise InvalidArgument("tensor must be contiguous")
        return C.c_void_p(buf.data_ptr()), buf
    arr = np.ascontiguousarray(buf)
    return C.c_void_p(arr.ctypes.data), arr


def _stream(stream):
    if stream is None:
        try:
            import torch

            if torch.cuda.is_available():
                return C.c_void_p(torch.cuda.current_stream().cuda_stream)
        except Exception:
            pass
        return None
    if hasattr(stream, "cuda_stream"):
        return C.c_void_p(stream.cuda_stream)
    return C.c_void_p(int(stream))


@dataclass
class EngineGeometry:
    n_seqs: int
    n_layers: int
    n_kv_heads: int
    head_dim: int
    dtype: int = DTYPE_BF16
    granularity: int = Granularity.PER_KV_HEAD
    capacity: int = 0
    max_pages_per_table: int = 0
    device: int = 0


class PagedEvictionEngine:
    """One rank's PagePool + every BlockTable + the eviction policy, in HBM."""

    def __init__(self, geometry: EngineGeometry, policy: PolicyConfig | None = None):
        policy = policy or PolicyConfig()
        if policy.kind not in (PolicyKind.PagedEviction, PolicyKind.FullCache):
            raise InvalidArgument(f"device engine implements paged-eviction and full, not {to_string(policy.kind)}")
        self.lib = _lib.load()
        self.geometry = geometry
        self.policy = policy
        cfg = _lib.PeConfig(
            n_seqs=geometry.n_seqs, n_layers=geometry.n_layers, n_kv_heads=geometry.n_kv_heads,
            head_dim=geometry.head_dim, granularity=int(geometry.granularity),
            page_size=policy.page_size, cache_budget=policy.cache_budget, dtype=geometry.dtype,
            policy=int(policy.kind), capacity=geometry.capacity,
            max_pages_per_table=geometry.max_pages_per_table, device=geometry.device)
        h = C.c_void_p()
        _check(self.lib.pe_engine_create(C.byref(cfg), C.byref(h)))
        self.h = h
        info = self.info()
        self.n_tables = info.n_tables
        self.tab_heads = info.tab_heads
        self.width = info.width
        self.capacity = info.capacity
        self.max_pages = info.max_pages
        self.B = info.page_size
        self.C = info.cache_budget

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.pe_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------- operations
    def table_id(self, seq: int, layer: int, head: int = 0) -> int:
        return (seq * self.geometry.n_layers + layer) * self.tab_heads + head

    def prefill_compress(self, layer, k, v, cu_seqlens, seq_begin=0, evicted_counts=None,
                         stream=None):
        """EvictionPolicy::prefill_compress + append of the survivors for every
        table of `layer` (policy.cpp:54-63, 90-101; block_table.cpp:10-19).
        Returns the per-table evicted count (launch order) when requested."""
        cu = np.ascontiguousarray(cu_seqlens, dtype=np.int32)
        want = evicted_counts is True
        if want:
            evicted_counts = np.zeros((cu.size - 1) * self.tab_heads, dtype=np.int32)
        pk, ka = _ptr(k)
        pv, va = _ptr(v)
        pe_, ea = _ptr(evicted_counts)
        _check(self.lib.pe_prefill_prune_pack(self.h, layer, pk, pv, C.c_void_p(cu.ctypes.data),
                                              seq_begin, cu.size - 1, pe_, _stream(stream)))
        if want:
            self.sync()
            return evicted_counts
        return None

    def append_token(self, layer_begin, n_layers, k_rows, v_rows, positions, stream=None):
        """BlockTable::append_token for every table of the layers (block_table.cpp:10-19)."""
        pos = positions if hasattr(positions, "data_ptr") else np.ascontiguousarray(positions, dtype=np.int64)
        pk, ka = _ptr(k_rows)
        pv, va = _ptr(v_rows)
        pp, pa = _ptr(pos)
        _check(self.lib.pe_decode_append(self.h, layer_begin, n_layers, pk, pv, pp, _stream(stream)))

    def evict(self, layer_begin, n_layers, step=0, mode=ScoreMode.RECOMPUTE, victims=None,
              stream=None):
        """PagedEvictionPolicy::evict for every table (policy.cpp:143-155).
        With victims=True returns the logical page index evicted per table
        (launch order) or -1."""
        want = victims is True
        if want:
            victims = np.zeros(n_layers * self.geometry.n_seqs * self.tab_heads, dtype=np.int32)
        pv, va = _ptr(victims)
        _check(self.lib.pe_decode_evict(self.h, layer_begin, n_layers, step, int(mode), pv,
                                        _stream(stream)))
        if want:
            self.sync()
            return victims
        return None

    def decode_step(self, layer_begin, n_layers, k_rows, v_rows, positions, step,
                    mode=ScoreMode.RECOMPUTE, victims=None, stream=None):
        """EvictionPolicy::decode_step (policy.cpp:65-70): append then evict."""
        self.append_token(layer_begin, n_layers, k_rows, v_rows, positions, stream)
        return self.evict(layer_begin, n_layers, step, mode, victims, stream)

    def attend(self, layer, q, out, n_q_heads, stream=None):
        """attend per query head over the pruned tables (attention.cpp:15-99)."""
        pq, qa = _ptr(q)
        po, oa = _ptr(out)
        _check(self.lib.pe_paged_decode_attention(self.h, layer, pq, po, n_q_heads, _stream(stream)))
        return out

    def sync(self) -> None:
        _check(self.lib.pe_sync(self.h))

    # ------------------------------------------------------------- readback
    def info(self) -> _lib.PeInfo:
        out = _lib.PeInfo()
        _check(self.lib.pe_get_info(self.h, C.byref(out)))
        return out

    def stats(self) -> _lib.PeStats:
        out = _lib.PeStats()
        _check(self.lib.pe_get_stats(self.h, C.byref(out)))
        return out

    def evict_tokens(self, layer_begin, n_layers, rule, arg, newest_positions, victims=None, stream=None):
        """Decode step of the StreamingLLM / InvKeyL2 / KeyDiff baselines over
        every table of the layer range, after the step's append_token
        (pe_decode_evict_tokens; policy.cpp:184-283): tables over budget evict
        one token by `rule`. With victims=True returns the evicted position
        per table (launch order) or -1."""
        want = victims is True
        if want:
            victims = np.zeros(n_layers * self.geometry.n_seqs * self.tab_heads, dtype=np.int64)
        pn, na = _ptr(newest_positions)
        pv, va = _ptr(victims)
        _check(self.lib.pe_decode_evict_tokens(self.h, layer_begin, n_layers, int(rule), int(arg), pn, pv,
                                               _stream(stream)))
        if want:
            self.sync()
            return victims
        return None

    def page_holes(self) -> np.ndarray:
        """Per page u64 mask of evicted slots (unstructured eviction)."""
        out = np.zeros(self.capacity, dtype=np.uint64)
        _check(self.lib.pe_read_page_holes(self.h, 0, self.capacity, C.c_void_p(out.ctypes.data)))
        return out

    def step_log(self, layer_begin, n_layers, victims=None, out=None, stream=None):
        """Engine-owned StepRecord fields of every table of the layer range
        after the preceding evict / decode_step (pe_step_log_capture):
        [n, 4] int32 rows (retained_len, page_count, newest_fill, victim), in
        launch order. victims: the device array given to that evict, or None
        for the engine's copy. Returns a host array unless `out` (device) is
        given; see steplog.step_records for the StepRecords."""
        n = n_layers * self.geometry.n_seqs * self.tab_heads
        host = out is None
        if host:
            out = np.zeros((n, 4), dtype=np.int32)
        pv, va = _ptr(victims)
        po, oa = _ptr(out)
        _check(self.lib.pe_step_log_capture(self.h, layer_begin, n_layers, pv, po, _stream(stream)))
        if host:
            self.sync()
        return out

    def check_invariants(self) -> dict:
        """Device-side structural invariants of every table and the pool
        (pe_check_invariants; selfcheck.cpp:19-75): returns the counts,
        `violations` == 0 when everything holds."""
        out = _lib.PeInvariants()
        _check(self.lib.pe_check_invariants(self.h, C.byref(out)))
        return {name: int(getattr(out, name)) for name, _ in _lib.PeInvariants._fields_}

    def device_view(self) -> _lib.PeDeviceView:
        out = _lib.PeDeviceView()
        _check(self.lib.pe_get_device_view(self.h, C.byref(out)))
        return out

    def tables(self):
        bt = np.zeros((self.n_tables, self.max_pages), dtype=np.int32)
        npg = np.zeros(self.n_tables, dtype=np.int32)
        nf = np.zeros(self.n_tables, dtype=np.int32)
        rt = np.zeros(self.n_tables, dtype=np.int32)
        _check(self.lib.pe_read_tables(self.h, C.c_void_p(bt.ctypes.data), C.c_void_p(npg.ctypes.data),
                                       C.c_void_p(nf.ctypes.data), C.c_void_p(rt.ctypes.data)))
        return bt, npg, nf, rt

    def free_list(self) -> np.ndarray:
        out = np.zeros(max(self.capacity, 1), dtype=np.int32)
        n = C.c_int32()
        _check(self.lib.pe_read_free_list(self.h, C.c_void_p(out.ctypes.data), C.byref(n)))
        return out[: n.value].copy()

    def free_count(self) -> int:
        """PagePool::free_count (page_pool.cpp:40-43)"""
        return int(self.info().free_pages)

    def allocated(self) -> int:
        """PagePool::allocated (page_pool.cpp:45-48)"""
        return self.capacity - self.free_count()

    def positions(self, page_begin=0, n_pages=None, scores=False):
        n_pages = self.capacity - page_begin if n_pages is None else n_pages
        pos = np.zeros((n_pages, self.B), dtype=np.int32)
        ts = np.zeros((n_pages, self.B), dtype=np.float64) if scores else None
        ps = np.zeros(n_pages, dtype=np.float64) if scores else None
        _check(self.lib.pe_read_positions(
            self.h, page_begin, n_pages, C.c_void_p(pos.ctypes.data),
            C.c_void_p(ts.ctypes.data) if scores else None,
            C.c_void_p(ps.ctypes.data) if scores else None))
        return (pos, ts, ps) if scores else pos

    def pages(self, page_begin=0, n_pages=None) -> np.ndarray:
        n_pages = self.capacity - page_begin if n_pages is None else n_pages
        dt = np.uint16 if self.geometry.dtype == DTYPE_BF16 else np.float32
        out = np.zeros((n_pages, 2, self.B, self.width), dtype=dt)
        _check(self.lib.pe_read_pages(self.h, page_begin, n_pages, C.c_void_p(out.ctypes.data)))
        return out

    def state(self, with_pages=True) -> dict:
        """Engine state in the oracle's layout (tests/harness.py)."""
        bt, npg, nf, rt = self.tables()
        pos, ts, ps = self.positions(scores=True)
        st = dict(block_table=bt, num_pages=npg, newest_fill=nf, retained=rt,
                  free_stack=self.free_list(), positions=pos, token_scores=ts, page_scores=ps)
        if with_pages:
            st["pages"] = self.pages()
        return st

    # per-table accessors (block_table.hpp:61-91)
    def page_count(self, t: int) -> int:
        return int(self.tables()[1][t])

    def retained_len(self, t: int) -> int:
        return int(self.tables()[3][t])

    def physical_id_at(self, t: int, logical_index: int) -> int:
        bt, npg, _, _ = self.tables()
        if logical_index >= npg[t]:
            raise IndexOutOfRange(f"logical page index {logical_index} out of range")
        return int(bt[t, logical_index])

    def retained_positions(self, t: int) -> np.ndarray:
        bt, npg, nf, _ = self.tables()
        pos = self.positions()
        out = []
        for j in range(npg[t]):
            fill = self.B if j < npg[t] - 1 else nf[t]
            out.append(pos[bt[t, j], :fill])
        return np.concatenate(out) if out else np.zeros(0, np.int32)
