"""CPU-side checks of the drop-in boundary: the C-ABI library builds, loads
without a GPU, exports every symbol include/pe.h declares, and fails
loudly (PE_NO_DEVICE) instead of falling back to the CPU."""
import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "pe.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pe_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_path():
    fns = declared_functions()
    for f in ("pe_engine_create", "pe_engine_destroy", "pe_prefill_prune_pack", "pe_decode_append",
              "pe_decode_evict", "pe_decode_step", "pe_paged_decode_attention", "pe_sync",
              "pe_read_tables", "pe_read_free_list", "pe_read_positions", "pe_read_pages"):
        assert f in fns


def test_library_exports_every_declared_symbol(engine_lib):
    for name in declared_functions():
        assert hasattr(engine_lib, name), f"libpe_b200.so does not export {name}"


def test_binding_covers_header():
    from paper_2509_04377_b200 import _lib

    assert set(_lib.SIGNATURES) == set(declared_functions())


def test_no_cpu_fallback(engine_lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2509_04377_b200 import _lib

    cfg = _lib.PeConfig(n_seqs=1, n_layers=1, n_kv_heads=1, head_dim=8, granularity=0,
                        page_size=16, cache_budget=64, dtype=0, policy=0, capacity=0,
                        max_pages_per_table=0, device=0)
    h = C.c_void_p()
    st = engine_lib.pe_engine_create(C.byref(cfg), C.byref(h))
    assert st == 31  # PE_NO_DEVICE
    assert b"device" in engine_lib.pe_last_error()


def test_config_validation_precedes_device_check(engine_lib):
    from paper_2509_04377_b200 import _lib

    cfg = _lib.PeConfig(n_seqs=1, n_layers=1, n_kv_heads=1, head_dim=8, granularity=0,
                        page_size=16, cache_budget=1000, dtype=0, policy=0, capacity=0,
                        max_pages_per_table=0, device=0)
    h = C.c_void_p()
    assert engine_lib.pe_engine_create(C.byref(cfg), C.byref(h)) == 9  # BudgetInvalid
    cfg.cache_budget = 8
    assert engine_lib.pe_engine_create(C.byref(cfg), C.byref(h)) == 9
    cfg.cache_budget = 64
    cfg.head_dim = 3  # 12-byte rows
    assert engine_lib.pe_engine_create(C.byref(cfg), C.byref(h)) == 20


def test_policy_mirror():
    import paper_2509_04377_b200 as pe

    for kind in pe.PolicyKind:
        assert pe.parse_policy_kind(pe.to_string(kind)) == kind
    assert pe.parse_policy_kind("h2o") is None
    with pytest.raises(pe.BudgetInvalid):
        pe.PolicyConfig(cache_budget=1000).validate()
    with pytest.raises(pe.BudgetInvalid):
        pe.PolicyConfig(cache_budget=8).validate()
    pe.PolicyConfig(cache_budget=4096).validate()


def test_facade_library_exports_the_reference_api():
    """libpagedevict_b200.so (the C++ façade) exports the reference's
    pagedevict:: entry points and links the C-ABI engine."""
    import subprocess

    from paper_2509_04377_b200 import _build

    _build.build()
    lib = _build.FACADE_LIB
    assert lib.exists()
    syms = subprocess.run(["nm", "-DC", "--defined-only", str(lib)], capture_output=True, text=True).stdout
    for sym in ("pagedevict::PagePool::PagePool", "pagedevict::PagePool::allocate",
                "pagedevict::BlockTable::append_token", "pagedevict::BlockTable::free_page",
                "pagedevict::BlockTable::retained_positions", "pagedevict::EvictionPolicy::prefill_compress",
                "pagedevict::EvictionPolicy::decode_step", "pagedevict::make_policy",
                "pagedevict::attend(", "pagedevict::rank_tokens", "pagedevict::rank_pages",
                "pagedevict::score_pages", "pagedevict::memory_bytes", "pagedevict::PolicyConfig::validate"):
        assert sym in syms, sym
    deps = subprocess.run(["ldd", str(lib)], capture_output=True, text=True).stdout
    assert "libpe_b200.so" in deps
    C.CDLL(str(lib))  # loads without a GPU


def test_reference_unit_tests_compile_against_the_facade():
    """Drop-in at the source level: the reference's own unit tests for the
    cache-manager API and a reference-API-only program build unchanged
    against include/pagedevict/*.hpp + libpagedevict_b200.so (run on the GPU
    by tests/test_facade_gpu.py)."""
    from pathlib import Path

    import pytest

    if not Path("/root/reference/proj").exists():
        pytest.skip("reference tree not present (GPU box): binaries are prebuilt")
    from tests.cpp import build_conformance as bc

    out = bc.build_reference_conformance()
    assert out is not None and out.exists()
    b200, ref = bc.build_scenario()
    assert b200.exists() and ref is not None and ref.exists()
    # every hot-path header the reference tests include resolves to the façade
    for h in ("page_pool", "block_table", "policy", "importance", "attention", "kv_vector", "page", "errors"):
        assert '#include "pe/pagedevict.hpp"' in (ROOT / "include" / "pagedevict" / f"{h}.hpp").read_text()
