"""Per-phase clock64 timing of the CTA select (debug build ab/libpe_b200_dbg.so)."""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
os.environ["PE_LIB"] = os.path.abspath("ab/libpe_b200_dbg.so")
import paper_2509_04377_b200 as pe
from paper_2509_04377_b200 import _lib
lib = _lib.load()
S, H, d, L, C_ = 16, 8, 128, 32768, 4096
eng = pe.PagedEvictionEngine(pe.EngineGeometry(n_seqs=S, n_layers=2, n_kv_heads=H, head_dim=d, dtype=1),
                             pe.PolicyConfig(cache_budget=C_, page_size=16))
dbg = torch.zeros(S * H * 8, dtype=torch.int64, device="cuda")
lib.pe_debug_set_select_timing.argtypes = [C.c_void_p]
k = torch.randn((S * L, H, d), device="cuda").to(torch.bfloat16)
v = torch.randn((S * L, H, d), device="cuda").to(torch.bfloat16)
cu = np.arange(S + 1, dtype=np.int32) * L
os.environ["PE_PREFILL_WAVES"] = "1"
eng.prefill_compress(0, k, v, cu); eng.sync()
lib.pe_debug_set_select_timing(C.c_void_p(dbg.data_ptr()))
eng.prefill_compress(1, k, v, cu); eng.sync()
t = dbg.view(S * H, 8).cpu().numpy().astype(np.float64)
ph = np.diff(t[:, :7], axis=1)
names = ["sample+sort", "load+window", "radix", "sweep_count", "sweep_emit", "metadata"]
print("cycles per phase (median over", ph.shape[0], "CTAs):")
for i, n in enumerate(names):
    print(f"  {n:12s} {np.median(ph[:, i]):10.0f}")
print("  total       ", np.median(t[:, 6] - t[:, 0]))
