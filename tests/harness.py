"""Shared parity-test helpers: seeded inputs, a replay of engine launches
through the REAL reference objects in the canonical batched order, and
state comparison (block tables, free list, positions, page bytes).

The engine state dict layout (produced by ``oracle.OracleEngine`` and by the
CUDA engine's readback) is:

    block_table [n_tables, max_pages] int32, num_pages / newest_fill /
    retained [n_tables] int32, free_stack [top] int32 (bottom..top),
    positions [cap, B] int32, pages [cap, 2, B, w] (float32 or bf16 bits).
"""
from __future__ import annotations

import numpy as np

import oracle


def random_kv(rng: np.random.Generator, shape, dtype: int):
    """Gaussian N(0,1) values in the engine dtype. Returns (engine array,
    exact float32 view)."""
    x = rng.standard_normal(shape, dtype=np.float32)
    if dtype == oracle.BF16:
        bits = oracle.f32_to_bf16_bits(x)
        return bits, oracle.bf16_bits_to_f32(bits)
    return x, x


def grid_kv(rng: np.random.Generator, shape, dtype: int, levels: int = 3):
    """Tie-heavy lattice inputs: small integers / 8 (exact in bf16 and
    float32). Many tokens share identical norms and therefore identical
    scores, exercising the (score, position) tie rules."""
    x = (rng.integers(-levels, levels + 1, size=shape) / 8.0).astype(np.float32)
    if dtype == oracle.BF16:
        bits = oracle.f32_to_bf16_bits(x)
        return bits, oracle.bf16_bits_to_f32(bits)
    return x, x


def as_f32(a: np.ndarray) -> np.ndarray:
    return oracle.bf16_bits_to_f32(a) if a.dtype == np.uint16 else a.astype(np.float32)


class RefReplay:
    """Drives one reference BlockTable + PagedEviction policy per engine table
    in the engine's canonical order:

    * prefill launch: tables in ascending id, each prefill_compress + append;
    * decode launch: decode_step on the tables whose append pops a page first
      (ascending id), then on the rest (ascending id) — i.e. all free-list
      pops before all pushes (exact for B >= 2).
    """

    def __init__(self, ref: oracle.Reference, *, n_seqs, n_layers, n_tab_heads, width,
                 page_size, budget, capacity, kind=oracle.PAGED_EVICTION):
        self.n_seqs, self.n_layers, self.H = n_seqs, n_layers, n_tab_heads
        self.B, self.C, self.w = page_size, budget, width
        self.n_tables = n_seqs * n_layers * n_tab_heads
        self.sess = ref.session(capacity, page_size, budget, self.n_tables, width, kind)
        self.kind = kind

    def tid(self, s, l, h):
        return (s * self.n_layers + l) * self.H + h

    def prefill(self, layer, k32, v32, cu, seq_begin=0):
        """k32/v32: float32 [tokens, H, w]. Returns evicted positions per
        launch table (list, launch order)."""
        out = []
        for s in range(len(cu) - 1):
            for h in range(self.H):
                t = self.tid(seq_begin + s, layer, h)
                ev = self.sess.prefill(t, k32[cu[s]:cu[s + 1], h], v32[cu[s]:cu[s + 1], h])
                out.append(ev)
        return out

    def decode(self, layer_begin, n_layers, k32, v32, positions, step):
        """k32/v32 float32 [n_layers, n_seqs, H, w]. Returns victims in launch
        order (logical index or -1)."""
        order = []
        for s in range(self.n_seqs):
            for li in range(n_layers):
                for h in range(self.H):
                    order.append((s, li, h))
        def pops(item):
            s, li, h = item
            t = self.tid(s, layer_begin + li, h)
            n = self.sess.page_count(t)
            return n == 0 or self._newest_fill(t) == self.B
        popping = [it for it in order if pops(it)]
        rest = [it for it in order if not pops(it)]
        victims = {}
        for s, li, h in popping + rest:
            t = self.tid(s, layer_begin + li, h)
            kind, idx = self.sess.decode_step(t, k32[li, s, h], v32[li, s, h],
                                              int(positions[s]), step)
            victims[(s, li, h)] = idx if kind == 2 else -1
        return np.array([victims[it] for it in order], dtype=np.int32)

    def _newest_fill(self, t):
        n = self.sess.page_count(t)
        r = self.sess.retained_len(t)
        return r - (n - 1) * self.B  # every non-newest page is full

    def attend(self, layer, q32, G):
        """q32 [n_seqs, H*G, d] -> out float32, one attend per query head
        (head_count = 1) on its KV head's table."""
        out = np.zeros_like(q32, dtype=np.float32)
        for s in range(self.n_seqs):
            for h in range(self.H):
                t = self.tid(s, layer, h)
                for g in range(G):
                    out[s, h * G + g] = self.sess.attend(t, q32[s, h * G + g], 1, self.w)
        return out


def compare_with_reference(rep: RefReplay, st: dict, tables=None, check_pages=True):
    """Asserts bit-exact equality of an engine state dict with the reference
    objects of a RefReplay."""
    B = rep.B
    tables = range(rep.n_tables) if tables is None else tables
    pages = st["pages"]
    for t in tables:
        r = rep.sess.read_table(t, with_data=check_pages)
        n = int(st["num_pages"][t])
        assert n == len(r["phys"]), f"table {t}: page_count {n} != ref {len(r['phys'])}"
        assert int(st["retained"][t]) == len(r["positions"]), f"table {t}: retained"
        np.testing.assert_array_equal(st["block_table"][t, :n], r["phys"],
                                      err_msg=f"table {t}: block_table")
        if n:
            assert int(st["newest_fill"][t]) == int(r["fills"][-1]), f"table {t}: newest fill"
            assert np.all(r["fills"][:-1] == B)
        pos, ks, vs = [], [], []
        for j in range(n):
            pid = int(st["block_table"][t, j])
            fill = B if j < n - 1 else int(st["newest_fill"][t])
            pos.append(st["positions"][pid, :fill])
            if check_pages:
                ks.append(as_f32(pages[pid, 0, :fill]))
                vs.append(as_f32(pages[pid, 1, :fill]))
        if n:
            np.testing.assert_array_equal(np.concatenate(pos), r["positions"],
                                          err_msg=f"table {t}: positions")
            if check_pages:
                np.testing.assert_array_equal(np.concatenate(ks), r["keys"],
                                              err_msg=f"table {t}: key bytes")
                np.testing.assert_array_equal(np.concatenate(vs), r["values"],
                                              err_msg=f"table {t}: value bytes")
    np.testing.assert_array_equal(st["free_stack"], rep.sess.mirror_free_list(),
                                  err_msg="free list")


def oracle_state(eng: oracle.OracleEngine) -> dict:
    return dict(block_table=eng.block_table(), num_pages=eng.num_pages(),
                newest_fill=eng.newest_fill(), retained=eng.retained(),
                free_stack=eng.free_stack(), positions=eng.positions(), pages=eng.pages(),
                page_scores=eng.page_scores())


def compare_states(a: dict, b: dict, n_tables: int, B: int, check_pages=True, what=""):
    """Bit-exact comparison of two engine state dicts (e.g. CUDA vs oracle)."""
    for key in ("num_pages", "newest_fill", "retained"):
        np.testing.assert_array_equal(a[key], b[key], err_msg=f"{what}{key}")
    np.testing.assert_array_equal(a["free_stack"], b["free_stack"], err_msg=f"{what}free list")
    for t in range(n_tables):
        n = int(a["num_pages"][t])
        np.testing.assert_array_equal(a["block_table"][t, :n], b["block_table"][t, :n],
                                      err_msg=f"{what}block_table[{t}]")
        for j in range(n):
            pid = int(a["block_table"][t, j])
            fill = B if j < n - 1 else int(a["newest_fill"][t])
            np.testing.assert_array_equal(a["positions"][pid, :fill], b["positions"][pid, :fill],
                                          err_msg=f"{what}positions page {pid}")
            if check_pages:
                np.testing.assert_array_equal(a["pages"][pid, :, :fill], b["pages"][pid, :, :fill],
                                              err_msg=f"{what}page bytes {pid}")


def compare_states_vectorized(a: dict, b: dict, B: int, check_pages=True, what=""):
    """compare_states for large engines (10^5+ tables): the same bit-exact
    checks, vectorised over every mapped (table, logical page) slot."""
    for key in ("num_pages", "newest_fill", "retained"):
        np.testing.assert_array_equal(a[key], b[key], err_msg=f"{what}{key}")
    np.testing.assert_array_equal(a["free_stack"], b["free_stack"], err_msg=f"{what}free list")
    npg = a["num_pages"].astype(np.int64)
    cols = np.arange(a["block_table"].shape[1])[None, :]
    mapped = cols < npg[:, None]
    np.testing.assert_array_equal(a["block_table"][mapped], b["block_table"][mapped],
                                  err_msg=f"{what}block tables")
    pids = a["block_table"][mapped].astype(np.int64)
    # fill of each mapped page: B except the newest
    is_newest = (cols == (npg[:, None] - 1))[mapped]
    fill = np.where(is_newest, np.repeat(a["newest_fill"], npg), B)
    slot_ok = np.arange(B)[None, :] < fill[:, None]
    np.testing.assert_array_equal(np.where(slot_ok, a["positions"][pids], 0),
                                  np.where(slot_ok, b["positions"][pids], 0), err_msg=f"{what}positions")
    if check_pages:
        m = slot_ok[:, None, :, None]
        np.testing.assert_array_equal(np.where(m, a["pages"][pids], 0), np.where(m, b["pages"][pids], 0),
                                      err_msg=f"{what}page bytes")
