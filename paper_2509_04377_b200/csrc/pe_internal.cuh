// Internal device-side definitions of the B200 PagedEviction engine.
//
// HBM layout:
//   pages        [capacity][2 (K,V)][B][row_pitch]   row_pitch = round_up(w*elt, 16)
//   positions    [capacity][B] int32
//   token_scores [capacity][B] double   (cached S of every written slot)
//   page_scores  [capacity] double      (mean S of a full page, set when it fills)
//   block_table  [n_tables][max_pages] int32, num_pages/newest_fill/retained [n_tables]
//   stack        [capacity] int32 + top   (LIFO free list, page_pool.cpp:18-38)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "pe/pe.h"

namespace pe {

constexpr int kWarp = 32;
constexpr int kChunkBytes = 256;                 // column chunk streamed per row per stage
constexpr int kStageRowPitch = kChunkBytes + 16; // padded smem row: conflict-free lane-per-row LDS.128
constexpr int kRowsPerSet = 32;                  // one row per lane
constexpr int kStageBytes = kRowsPerSet * kStageRowPitch;  // 8704 B
constexpr double kNormEps = 1e-12;               // kNormEpsilon, importance.hpp:17

struct DevState {
    uint8_t* pages;
    int32_t* positions;
    double* token_scores;
    double* page_scores;
    int32_t* block_table;
    int32_t* num_pages;
    int32_t* newest_fill;
    int32_t* retained;
    int32_t* stack;
    int32_t* top;
    int32_t* status;
    unsigned long long* evict_count;
    int32_t capacity, B, C, w, pitch, row_bytes, max_pages, n_tables;
    int32_t n_seqs, n_layers, tab_heads, dtype, policy;
};

// Per-launch control block written by the plan kernels.
struct LaunchCtl {
    int32_t abort;      // 1: the launch is a no-op (status set)
    int32_t pop_base;   // stack top before this launch's pops
    int32_t push_base;  // stack top before this launch's pushes
    int32_t count;      // number of flagged tables (evict work items)
};

// Launch table set: decode launches cover every sequence for layers
// [layer_begin, layer_begin+n_layers); index i enumerates (seq, layer, head)
// seq-major, which is ascending table id.
struct TableSet {
    int32_t layer_begin, n_layers;
    __host__ __device__ int32_t size(const DevState& s) const { return s.n_seqs * n_layers * s.tab_heads; }
    __host__ __device__ int32_t table(const DevState& s, int32_t i) const {
        const int32_t h = i % s.tab_heads;
        const int32_t rest = i / s.tab_heads;
        const int32_t li = rest % n_layers;
        const int32_t seq = rest / n_layers;
        return (seq * s.n_layers + layer_begin + li) * s.tab_heads + h;
    }
    // row index of launch table i in an input laid out [n_layers][n_seqs][tab_heads]
    __host__ __device__ int64_t input_row(const DevState& s, int32_t i) const {
        const int32_t h = i % s.tab_heads;
        const int32_t rest = i / s.tab_heads;
        const int32_t li = rest % n_layers;
        const int32_t seq = rest / n_layers;
        return ((int64_t)li * s.n_seqs + seq) * s.tab_heads + h;
    }
};

__device__ __forceinline__ void set_status(int32_t* status, int32_t code) {
    atomicCAS(status, 0, code);
}

// ------------------------------------------------------------------ async copy
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ uint4 ld_shared_v4(const void* p) {
    uint4 r;
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(p));
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "r"(s));
    return r;
}

// ------------------------------------------------------------------ exact fp64 sum of squares
//
// The reference sums x*x in double, in index order (l2_norm,
// kv_vector.hpp:15-21). Every lane owns one row and sums it sequentially,
// so the result is bit-identical. Fast path: the element is turned into a
// double by integer ops (no F2F conversion) pre-scaled by 2^-384, so x^2 is
// scaled by 2^-768 — an exact power-of-two scaling that cannot change any
// rounding as long as every value stays a normal double, which holds for
// |x| >= 2^-60. Rows holding any element below that (zeros, subnormals,
// tiny values) are flagged and recomputed by the plain exact loop.

// bf16 pair -> two scaled doubles' high words; updates the packed-u16 minimum
// of |x| bit patterns used by the range check.
__device__ __forceinline__ void bf16x2_to_scaled(uint32_t w, double& d0, double& d1, uint32_t& mn) {
    const uint32_t a = w & 0x7FFF7FFFu;
    uint32_t m;
    asm("min.u16x2 %0, %1, %2;" : "=r"(m) : "r"(mn), "r"(a));
    mn = m;
    const uint32_t h0 = ((a << 13) & 0x0FFFE000u) | 0x20000000u;
    const uint32_t h1 = ((a >> 3) & 0x0FFFE000u) | 0x20000000u;
    d0 = __hiloint2double(static_cast<int>(h0), 0);
    d1 = __hiloint2double(static_cast<int>(h1), 0);
}

// fp32 -> scaled double; updates the minimum |x| bit pattern.
__device__ __forceinline__ double f32_to_scaled(uint32_t b, uint32_t& mn) {
    const uint32_t a = b & 0x7FFFFFFFu;
    mn = min(mn, a);
    const uint32_t hi = (a >> 3) | 0x20000000u;
    const uint32_t lo = a << 29;
    return __hiloint2double(static_cast<int>(hi), static_cast<int>(lo));
}

// 2^768 as a double (exponent field 1791).
__device__ __forceinline__ double two_pow_768() { return __hiloint2double(0x6FF00000, 0); }

// |x| >= 2^-60 thresholds on the bit patterns: bf16 exponent field >= 67
// (67 << 7 = 0x2180 per u16 lane), fp32 exponent field >= 67 (67 << 23).
constexpr uint32_t kBf16MinBits = 0x2180u;
constexpr uint32_t kF32MinBits = 67u << 23;

__device__ __forceinline__ bool bf16_range_ok(uint32_t mn) {
    return (mn & 0xFFFFu) >= kBf16MinBits && (mn >> 16) >= kBf16MinBits;
}

// Plain exact reference loop (slow path and single rows).
__device__ __forceinline__ double row_sumsq_exact(const uint8_t* row, int w, int dtype) {
    double acc = 0.0;
    if (dtype == PE_DTYPE_BF16) {
        const uint16_t* p = reinterpret_cast<const uint16_t*>(row);
        for (int i = 0; i < w; ++i) {
            const double x = static_cast<double>(__uint_as_float(static_cast<uint32_t>(p[i]) << 16));
            acc = fma(x, x, acc);
        }
    } else {
        const float* p = reinterpret_cast<const float*>(row);
        for (int i = 0; i < w; ++i) {
            const double x = static_cast<double>(p[i]);
            acc = fma(x, x, acc);
        }
    }
    return acc;
}

// Accumulates one 16-byte piece (8 bf16 or 4 fp32 elements, index order)
// into the scaled accumulator. `valid_elems` < full only on the row tail.
__device__ __forceinline__ void accum_piece(const uint4 v, int dtype, int valid_elems, double& acc,
                                            uint32_t& mn) {
    const uint32_t wds[4] = {v.x, v.y, v.z, v.w};
    if (dtype == PE_DTYPE_BF16) {
        if (valid_elems >= 8) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                double d0, d1;
                bf16x2_to_scaled(wds[k], d0, d1, mn);
                acc = fma(d0, d0, acc);
                acc = fma(d1, d1, acc);
            }
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                double d0, d1;
                // mask the second element of the pair if it is past the row end
                uint32_t wv = wds[k];
                if (2 * k >= valid_elems) break;
                if (2 * k + 1 >= valid_elems) wv = (wv & 0xFFFFu) | 0x3F800000u;  // pad: 1.0 (in range), not summed
                bf16x2_to_scaled(wv, d0, d1, mn);
                acc = fma(d0, d0, acc);
                if (2 * k + 1 < valid_elems) acc = fma(d1, d1, acc);
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (k < valid_elems) {
                const double d = f32_to_scaled(wds[k], mn);
                acc = fma(d, d, acc);
            }
        }
    }
}

// ------------------------------------------------------------------ warp row streamer
//
// A warp processes a sequence of "row sets" of 32 rows (one row per lane).
// Rows are streamed in 256-byte column chunks through an NSTAGE-deep
// cp.async ring in shared memory (coalesced 16-byte global loads, padded
// smem rows so the lane-per-row reads are bank-conflict free). Each lane
// sums its own row sequentially in index order -> exact fp64 sum of squares.
//
// AddrFn: const uint8_t* addr(int set, int row)  (nullptr = row absent)
// DoneFn: void done(int set, double sumsq, bool present)  (called by every lane)
template <int NSTAGE, typename AddrFn, typename DoneFn>
__device__ __forceinline__ void warp_stream_sumsq(int n_sets, int row_bytes, int w, int dtype,
                                                  uint8_t* stage, AddrFn addr, DoneFn done) {
    const int lane = threadIdx.x & 31;
    const int nchunk = (row_bytes + kChunkBytes - 1) / kChunkBytes;
    const int n_items = n_sets * nchunk;
    const int elt = dtype == PE_DTYPE_BF16 ? 2 : 4;
    const int elems_per_piece = 16 / elt;

    // issue the cp.async loads of item `it` into stage slot it % NSTAGE
    auto issue = [&](int it) {
        if (it < n_items) {
            const int set = it / nchunk;
            const int c = it - set * nchunk;
            uint8_t* slot = stage + (it % NSTAGE) * kStageBytes;
            const int col0 = c * kChunkBytes;
            const int piece = lane & 15;
            const int col = col0 + piece * 16;
#pragma unroll 4
            for (int j = 0; j < 16; ++j) {
                const int row = 2 * j + (lane >> 4);
                const uint8_t* g = addr(set, row);
                if (g != nullptr && col < row_bytes) {
                    cp_async16(slot + row * kStageRowPitch + piece * 16, g + col);
                }
            }
        }
        cp_async_commit();
    };

#pragma unroll
    for (int p = 0; p < NSTAGE - 1; ++p) issue(p);

    double acc = 0.0;
    uint32_t mn = 0xFFFFFFFFu;
    for (int it = 0; it < n_items; ++it) {
        issue(it + NSTAGE - 1);
        cp_async_wait<NSTAGE - 1>();
        __syncwarp();
        const int set = it / nchunk;
        const int c = it - set * nchunk;
        const uint8_t* slot = stage + (it % NSTAGE) * kStageBytes + lane * kStageRowPitch;
        const uint8_t* my = addr(set, lane);
        if (my != nullptr) {
            const int bytes = min(kChunkBytes, row_bytes - c * kChunkBytes);
            const int pieces = (bytes + 15) / 16;
            const int elems_left = w - c * (kChunkBytes / elt);
            if (pieces == 16 && elems_left >= 16 * elems_per_piece) {
#pragma unroll 4
                for (int p = 0; p < 16; ++p) {
                    accum_piece(ld_shared_v4(slot + p * 16), dtype, elems_per_piece, acc, mn);
                }
            } else {
                for (int p = 0; p < pieces; ++p) {
                    const int valid = min(elems_per_piece, elems_left - p * elems_per_piece);
                    if (valid <= 0) break;
                    accum_piece(ld_shared_v4(slot + p * 16), dtype, valid, acc, mn);
                }
            }
        }
        __syncwarp();  // slot may be overwritten by the next issue
        if (c == nchunk - 1) {
            double r = 0.0;
            if (my != nullptr) {
                const bool ok = (dtype == PE_DTYPE_BF16) ? bf16_range_ok(mn) : (mn >= kF32MinBits);
                r = ok ? acc * two_pow_768() : row_sumsq_exact(my, w, dtype);
            }
            done(set, r, my != nullptr);
            acc = 0.0;
            mn = 0xFFFFFFFFu;
        }
    }
    cp_async_wait<0>();
    __syncwarp();
}

// S = ||V|| / max(||K||, eps) from the two sums of squares (importance.cpp:11-13).
__device__ __forceinline__ double token_score_from_sumsq(double k2, double v2) {
    const double kn = sqrt(k2);
    const double vn = sqrt(v2);
    return vn / fmax(kn, kNormEps);
}

// ------------------------------------------------------------------ warp/cta scans
__device__ __forceinline__ int warp_incl_scan(int v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

// Block-wide exclusive scan of one int per thread. `sm` needs 33 ints.
// Returns the exclusive prefix; *total receives the block total.
__device__ __forceinline__ int block_excl_scan(int v, int* sm, int* total) {
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    const int incl = warp_incl_scan(v);
    if (lane == 31) sm[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        int x = lane < nw ? sm[lane] : 0;
        const int xi = warp_incl_scan(x);
        if (lane < nw) sm[lane] = xi - x;
        if (lane == 31) sm[32] = xi;
    }
    __syncthreads();
    const int r = sm[wid] + incl - v;
    *total = sm[32];
    __syncthreads();
    return r;
}

}  // namespace pe
