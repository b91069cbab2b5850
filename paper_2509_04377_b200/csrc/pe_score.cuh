// Exact fp64 token scores, S = ||V|| / max(||K||, 1e-12), bit-identical to
// the reference (l2_norm: double sum of x*x in index order, kv_vector.hpp:15-21;
// token_importance, importance.cpp:11-13).
//
// Register-direct, two lanes per token: lane pair (2r, 2r+1) scores token r
// of a 16-token group. Lane q of the pair loads the 32-byte chunks q, q+2,
// ... of the token's K row and of its V row with 256-bit loads (one full
// sector per lane; every warp load instruction touches 16 rows x 64
// contiguous bytes; no shared memory).
//
// bf16 — exactness certificate instead of a serial chain. Each element is
// turned into a double by integer ops, pre-scaled by 2^-384 (bits: the bf16
// exponent+mantissa shifted into the double's high word, exponent bias
// +512), so x^2 is scaled by the exact power of two 2^-768. A square of a
// bf16 value has at most 16 significant bits and its lowest set bit is at
// or above 2*e_min - 1036 (e_min: smallest exponent field in the row, in
// the scaled domain). If the computed sum S_c of all squares satisfies
// S_c < 2^(2*e_min - 984) = 2^(lowest_bit + 52), then every partial sum in
// ANY order is an exactly representable multiple of 2^lowest_bit (proof in
// DESIGN.md §4), so the reference's sequential double sum equals the exact
// sum equals S_c: the lanes may use several independent DFMA chains and a
// shuffle reduction. Rows that fail the certificate (tiny or zero elements
// relative to the row's norm; ~0.3% of N(0,1) rows) take the plain
// sequential loop of the reference.
//
// fp32 — a square has up to 48 significant bits, so the certificate never
// holds for general data: lane 0 of the pair sums the K row and lane 1 the
// V row sequentially in index order (exact by construction).
#pragma once

#include "pe_internal.cuh"

namespace pe {

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(p));
    return r;
}

__device__ __forceinline__ void stg_v4(void* p, uint4 v) {
    *reinterpret_cast<uint4*>(p) = v;
}

// 256-bit streaming load (one full 32-byte sector per lane; LDG.E.256 on
// sm_100a) with an L2 prefetch of the enclosing 256-byte segment.
struct u32x8 {
    uint32_t w[8];
};
__device__ __forceinline__ u32x8 ldg256(const void* p) {
    u32x8 r;
    asm("ld.global.nc.L1::no_allocate.L2::256B.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]), "=r"(r.w[6]),
          "=r"(r.w[7])
        : "l"(p));
    return r;
}
__device__ __forceinline__ void stg256(void* p, const u32x8& v) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.w[0]), "r"(v.w[1]), "r"(v.w[2]),
                 "r"(v.w[3]), "r"(v.w[4]), "r"(v.w[5]), "r"(v.w[6]), "r"(v.w[7])
                 : "memory");
}

__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t m, uint32_t o) {
    uint32_t r;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(a), "r"(m), "r"(o));  // (a & m) | o
    return r;
}

__device__ __forceinline__ uint32_t min3_u32(uint32_t a, uint32_t b, uint32_t c) {
    return min(a, min(b, c));
}

// Two scaled doubles from one bf16x2 word; hmin tracks the smallest high word.
__device__ __forceinline__ void bf16x2_scaled(uint32_t w, double& d0, double& d1, uint32_t& hmin) {
    const uint32_t h0 = lop3_and_or(w << 13, 0x0FFFE000u, 0x20000000u);
    const uint32_t h1 = lop3_and_or(w >> 3, 0x0FFFE000u, 0x20000000u);
    hmin = min3_u32(hmin, h0, h1);
    d0 = __hiloint2double(static_cast<int>(h0), 0);
    d1 = __hiloint2double(static_cast<int>(h1), 0);
}

// Certificate check in the scaled domain (see the file comment). hmin is the
// smallest scaled high word: exponent field = bf16 exponent + 512.
__device__ __forceinline__ bool bf16_sum_certified(double s_scaled, uint32_t hmin) {
    const int e_field = static_cast<int>(hmin >> 20);  // bf16 exponent + 512
    if (e_field < 512 + 8) return false;               // zeros / subnormal-range squares
    const int thr_field = 2 * (e_field - 512) + 39;    // 2*e_min - 984 + 1023
    const double thr = __hiloint2double(thr_field << 20, 0);
    return s_scaled < thr;
}

static __device__ __noinline__ double row_sumsq_seq_bf16(const uint8_t* row, int w) {
    const uint16_t* p = reinterpret_cast<const uint16_t*>(row);
    double acc = 0.0;
    for (int i = 0; i < w; ++i) {
        const double x = static_cast<double>(__uint_as_float(static_cast<uint32_t>(__ldg(p + i)) << 16));
        acc = fma(x, x, acc);
    }
    return acc;
}

__device__ __forceinline__ double row_sumsq_seq_f32(const uint8_t* row, int w) {
    const float* p = reinterpret_cast<const float*>(row);
    double acc = 0.0;
    for (int i = 0; i < w; ++i) {
        const double x = static_cast<double>(__ldg(p + i));
        acc = fma(x, x, acc);
    }
    return acc;
}

// Sequential (index-order) sum of squares of one bf16 row by a lane pair,
// bit-identical to row_sumsq_seq_bf16: each lane reloads its 32-byte chunks
// (q, q+2, ...; cache hits, the row was just read) and the running sum is
// handed between the two lanes chunk by chunk, so the dependent chain is 16
// DFMAs per chunk instead of a load per element. For the rows the exactness
// certificate rejects (about 0.15 % of N(0,1) bf16 rows); both lanes of the
// pair must call it.
template <int CHUNKS>
__device__ __forceinline__ double pair_row_sumsq_seq_bf16(const uint8_t* row) {
    constexpr int NC = CHUNKS / 2;
    const int q = threadIdx.x & 1;
    const int base = (threadIdx.x & 31) & ~1;
    const unsigned pmask = 3u << base;
    u32x8 x[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) x[c] = ldg256(row + (2 * c + q) * 32);
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < CHUNKS; ++c) {
        if (q == (c & 1)) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t w = x[c >> 1].w[k];
                const double a = static_cast<double>(__uint_as_float(w << 16));
                const double b = static_cast<double>(__uint_as_float(w & 0xFFFF0000u));
                acc = fma(a, a, acc);
                acc = fma(b, b, acc);
            }
        }
        acc = __shfl_sync(pmask, acc, base + (c & 1));
    }
    return acc;
}

// This lane's share (32-byte chunks q, q+2, ...) of one bf16 row, already
// loaded: two DFMA chains + min tracking.
template <int NC>
__device__ __forceinline__ double pair_part_bf16(const u32x8 (&x)[NC], uint32_t& hmin) {
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            double d0, d1;
            bf16x2_scaled(x[c].w[k], d0, d1, hmin);
            a0 = fma(d0, d0, a0);
            a1 = fma(d1, d1, a1);
        }
    }
    return a0 + a1;
}

__device__ __forceinline__ u32x8 bf16_ones8() {
    u32x8 r;
#pragma unroll
    for (int k = 0; k < 8; ++k) r.w[k] = 0x3F803F80u;
    return r;
}

// Scores token `r = lane >> 1` given its K and V row pointers (both lanes of
// the pair pass the same pointers; `valid` false -> returns 0). Lane q of the
// pair loads the 32-byte chunks q, q+2, ... (one full sector per lane per
// 256-bit load; a warp load covers 16 rows x 64 contiguous bytes). When
// kdst / vdst are given the rows are also copied there from the same
// registers (decode append: one read serves the copy and the score).
// CHUNKS = row_bytes / 32 (even).
template <int CHUNKS>
__device__ __forceinline__ double pair_token_score_bf16(const uint8_t* krow, const uint8_t* vrow, bool valid,
                                                        uint8_t* kdst = nullptr, uint8_t* vdst = nullptr) {
    static_assert(CHUNKS % 2 == 0, "even chunk count");
    constexpr int NC = CHUNKS / 2;
    const int q = threadIdx.x & 1;
    uint32_t kmin = 0xFFFFFFFFu, vmin = 0xFFFFFFFFu;
    double kp = 0.0, vp = 0.0;
#pragma unroll
    for (int rv = 0; rv < 2; ++rv) {
        const uint8_t* row = rv ? vrow : krow;
        uint8_t* dst = rv ? vdst : kdst;
        u32x8 x[NC];
        if (valid) {
#pragma unroll
            for (int c = 0; c < NC; ++c) x[c] = ldg256(row + (2 * c + q) * 32);
            if (dst != nullptr) {
#pragma unroll
                for (int c = 0; c < NC; ++c) stg256(dst + (2 * c + q) * 32, x[c]);
            }
        } else {
#pragma unroll
            for (int c = 0; c < NC; ++c) x[c] = bf16_ones8();
        }
        if (rv == 0) kp = pair_part_bf16<NC>(x, kmin);
        else vp = pair_part_bf16<NC>(x, vmin);
    }
    kp += __shfl_xor_sync(0xFFFFFFFFu, kp, 1);
    vp += __shfl_xor_sync(0xFFFFFFFFu, vp, 1);
    kmin = min(kmin, __shfl_xor_sync(0xFFFFFFFFu, kmin, 1));
    vmin = min(vmin, __shfl_xor_sync(0xFFFFFFFFu, vmin, 1));
    const double s768 = two_pow_768();
    double k2 = kp * s768;
    double v2 = vp * s768;
    if (valid && !bf16_sum_certified(kp, kmin)) k2 = pair_row_sumsq_seq_bf16<CHUNKS>(krow);
    if (valid && !bf16_sum_certified(vp, vmin)) v2 = pair_row_sumsq_seq_bf16<CHUNKS>(vrow);
    const double S = pair_score_from_sumsq(k2, v2);  // all lanes: one sqrt each
    return valid ? S : 0.0;
}

// fp32: lane 0 of the pair sums the K row, lane 1 the V row, sequentially
// (and copies its row when a destination is given).
template <int CHUNKS>
__device__ __forceinline__ double pair_token_score_f32(const uint8_t* krow, const uint8_t* vrow, bool valid,
                                                       uint8_t* kdst = nullptr, uint8_t* vdst = nullptr) {
    const int q = threadIdx.x & 1;
    double acc = 0.0;
    if (valid) {
        const uint8_t* row = q ? vrow : krow;
        uint8_t* dst = q ? vdst : kdst;
#pragma unroll 2
        for (int c = 0; c < CHUNKS; ++c) {
            const u32x8 f = ldg256(row + c * 32);
            if (dst != nullptr) stg256(dst + c * 32, f);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const double x = static_cast<double>(__uint_as_float(f.w[k]));
                acc = fma(x, x, acc);
            }
        }
    }
    const double other = __shfl_xor_sync(0xFFFFFFFFu, acc, 1);
    if (!valid) return 0.0;
    const double k2 = q ? other : acc;
    const double v2 = q ? acc : other;
    return token_score_from_sumsq(k2, v2);
}

// Runtime-width fallbacks (rows of any multiple of 16 bytes).
__device__ __forceinline__ double pair_token_score_generic(const uint8_t* krow, const uint8_t* vrow, bool valid,
                                                           int w, int dtype, uint8_t* kdst = nullptr,
                                                           uint8_t* vdst = nullptr) {
    const int q = threadIdx.x & 1;
    double acc = 0.0;
    if (valid) {
        const uint8_t* row = q ? vrow : krow;
        uint8_t* dst = q ? vdst : kdst;
        const int bytes = w * (dtype == PE_DTYPE_BF16 ? 2 : 4);
        if (dst != nullptr) {
            for (int off = 0; off < bytes; off += 16)
                *reinterpret_cast<uint4*>(dst + off) = __ldg(reinterpret_cast<const uint4*>(row + off));
        }
        acc = dtype == PE_DTYPE_BF16 ? row_sumsq_seq_bf16(row, w) : row_sumsq_seq_f32(row, w);
    }
    const double other = __shfl_xor_sync(0xFFFFFFFFu, acc, 1);
    if (!valid) return 0.0;
    return token_score_from_sumsq(q ? other : acc, q ? acc : other);
}

// Row geometry the kernels are specialised for: (dtype, 16-byte pieces/row).
enum ScoreVariant : int {
    kScoreGeneric = 0,
    kScoreBf16x16 = 1,  // bf16, d = 128  (256-byte rows)
    kScoreBf16x8 = 2,   // bf16, d = 64
    kScoreF32x16 = 3,   // fp32, d = 64   (256-byte rows)
    kScoreF32x32 = 4,   // fp32, d = 128
};

__host__ __device__ inline int score_variant(int dtype, int row_bytes) {
    if (dtype == PE_DTYPE_BF16 && row_bytes == 256) return kScoreBf16x16;
    if (dtype == PE_DTYPE_BF16 && row_bytes == 128) return kScoreBf16x8;
    if (dtype == PE_DTYPE_F32 && row_bytes == 256) return kScoreF32x16;
    if (dtype == PE_DTYPE_F32 && row_bytes == 512) return kScoreF32x32;
    return kScoreGeneric;
}

template <int V>
__device__ __forceinline__ double pair_token_score(const uint8_t* krow, const uint8_t* vrow, bool valid, int w,
                                                   int dtype, uint8_t* kdst = nullptr, uint8_t* vdst = nullptr) {
    if constexpr (V == kScoreBf16x16) return pair_token_score_bf16<8>(krow, vrow, valid, kdst, vdst);
    else if constexpr (V == kScoreBf16x8) return pair_token_score_bf16<4>(krow, vrow, valid, kdst, vdst);
    else if constexpr (V == kScoreF32x16) return pair_token_score_f32<8>(krow, vrow, valid, kdst, vdst);
    else if constexpr (V == kScoreF32x32) return pair_token_score_f32<16>(krow, vrow, valid, kdst, vdst);
    else return pair_token_score_generic(krow, vrow, valid, w, dtype, kdst, vdst);
}

// Dispatch helper for kernel templates.
#define PE_SCORE_DISPATCH(variant, KERNEL_CALL)            \
    switch (variant) {                                     \
    case kScoreBf16x16: { constexpr int SV = kScoreBf16x16; KERNEL_CALL; } break; \
    case kScoreBf16x8: { constexpr int SV = kScoreBf16x8; KERNEL_CALL; } break;   \
    case kScoreF32x16: { constexpr int SV = kScoreF32x16; KERNEL_CALL; } break;   \
    case kScoreF32x32: { constexpr int SV = kScoreF32x32; KERNEL_CALL; } break;   \
    default: { constexpr int SV = kScoreGeneric; KERNEL_CALL; } break;           \
    }

}  // namespace pe
