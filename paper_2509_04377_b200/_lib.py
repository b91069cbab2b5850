"""ctypes binding of include/pe.h (libpe_b200.so).

Loading fails loudly: there is no CPU fallback for the PagedEviction hot path.
"""
from __future__ import annotations

import ctypes as C
import threading

from . import _build

_lock = threading.Lock()
_lib: C.CDLL | None = None

c_i32, c_i64, c_vp = C.c_int32, C.c_int64, C.c_void_p


class PeConfig(C.Structure):
    _fields_ = [(n, c_i32) for n in (
        "n_seqs", "n_layers", "n_kv_heads", "head_dim", "granularity", "page_size", "cache_budget",
        "dtype", "policy", "capacity", "max_pages_per_table", "device")]


class PeInfo(C.Structure):
    _fields_ = [(n, c_i32) for n in (
        "n_tables", "tab_heads", "width", "page_size", "cache_budget", "capacity", "max_pages",
        "dtype", "policy", "granularity", "row_pitch_bytes", "sm_count")] + [
        ("pool_bytes", c_i64), ("state_bytes", c_i64), ("free_pages", c_i32), ("pad_", c_i32)]


class PeStats(C.Structure):
    _fields_ = [(n, c_i64) for n in (
        "prefill_calls", "append_calls", "evict_calls", "attention_calls", "tokens_scored",
        "pages_evicted", "kernel_launches")]


class PeInvariants(C.Structure):
    _fields_ = [(n, c_i64) for n in (
        "tables_checked", "pages_mapped", "free_pages", "violations", "page_not_full",
        "retained_mismatch", "budget_violations", "position_order", "page_refcount")]


class PeDeviceView(C.Structure):
    _fields_ = [("pages", c_vp), ("block_table", c_vp), ("num_pages", c_vp),
                ("newest_fill", c_vp), ("retained", c_vp), ("positions", c_vp)]


# every symbol include/pe.h declares, with its signature
SIGNATURES = {
    "pe_abi_version": (c_i32, []),
    "pe_last_error": (C.c_char_p, []),
    "pe_status_string": (C.c_char_p, [C.c_int]),
    "pe_engine_create": (C.c_int, [C.POINTER(PeConfig), C.POINTER(c_vp)]),
    "pe_engine_destroy": (C.c_int, [c_vp]),
    "pe_prefill_prune_pack": (C.c_int, [c_vp, c_i32, c_vp, c_vp, c_vp, c_i32, c_i32, c_vp, c_vp]),
    "pe_decode_append": (C.c_int, [c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "pe_decode_evict": (C.c_int, [c_vp, c_i32, c_i32, c_i64, c_i32, c_vp, c_vp]),
    "pe_decode_step": (C.c_int, [c_vp, c_i32, c_i32, c_vp, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp]),
    "pe_paged_decode_attention": (C.c_int, [c_vp, c_i32, c_vp, c_vp, c_i32, c_vp]),
    "pe_sync": (C.c_int, [c_vp]),
    "pe_get_info": (C.c_int, [c_vp, C.POINTER(PeInfo)]),
    "pe_get_stats": (C.c_int, [c_vp, C.POINTER(PeStats)]),
    "pe_read_tables": (C.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pe_read_free_list": (C.c_int, [c_vp, c_vp, C.POINTER(c_i32)]),
    "pe_read_positions": (C.c_int, [c_vp, c_i32, c_i32, c_vp, c_vp, c_vp]),
    "pe_read_pages": (C.c_int, [c_vp, c_i32, c_i32, c_vp]),
    "pe_get_device_view": (C.c_int, [c_vp, C.POINTER(PeDeviceView)]),
    # table-granular API (the C++ façade's calls)
    "pe_table_append": (C.c_int, [c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pe_table_evict": (C.c_int, [c_vp, c_i32, c_vp, c_i32, c_i32, c_vp, c_vp]),
    "pe_table_free_page": (C.c_int, [c_vp, c_i32, c_i32, c_vp]),
    "pe_table_clear": (C.c_int, [c_vp, c_i32, c_vp]),
    "pe_table_attend": (C.c_int, [c_vp, c_i32, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp]),
    "pe_read_table": (C.c_int, [c_vp, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "pe_pool_allocate": (C.c_int, [c_vp, C.POINTER(c_i32)]),
    "pe_pool_release": (C.c_int, [c_vp, c_i32]),
    "pe_table_evict_token": (C.c_int, [c_vp, c_i32, c_i32, c_i64, c_i32, c_i64, c_vp, c_vp]),
    "pe_read_page_holes": (C.c_int, [c_vp, c_i32, c_i32, c_vp]),
    "pe_prompt_select": (C.c_int, [c_i32, c_i32, c_vp, c_i32, c_i32, c_vp, c_i32, c_vp]),
    "pe_check_invariants": (C.c_int, [c_vp, C.POINTER(PeInvariants)]),
    "pe_step_log_capture": (C.c_int, [c_vp, c_i32, c_i32, c_vp, c_vp, c_vp]),
    "pe_decode_evict_tokens": (C.c_int, [c_vp, c_i32, c_i32, c_i32, c_i64, c_vp, c_vp, c_vp]),
    "pe_probe_hbm": (C.c_int, [c_i32, c_i64, c_i32, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "pe_current_device": (C.c_int, [C.POINTER(c_i32)]),
}


def load() -> C.CDLL:
    """Builds (if stale) and loads libpe_b200.so. Raises if it cannot."""
    global _lib
    with _lock:
        if _lib is None:
            import os

            # PE_LIB: an alternative build of the same library (A/B timing runs)
            path = os.environ.get("PE_LIB") or _build.build()
            lib = C.CDLL(str(path))
            for name, (res, args) in SIGNATURES.items():
                if not hasattr(lib, name) and os.environ.get("PE_LIB"):
                    continue  # older A/B build without the newest entry points
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if lib.pe_abi_version() != 1:
                raise RuntimeError("libpe_b200.so ABI version mismatch")
            _lib = lib
    return _lib


def library_path() -> str:
    return str(_build.LIB)
