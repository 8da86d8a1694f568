// Warp-per-chunk building blocks for the ChunkSpec(8,8,8) fast paths (K1/K6).
//
// Register layout of one 8x8x8 chunk in a warp: lane l owns the two x-rows
//   row0 = (ly = l & 7, lz = 2*(l >> 3))   and   row1 = (ly, lz + 1),
// eight x-elements each.  Then
//   x neighbours are in-lane, y neighbours are one lane apart (shfl by 1,
//   width 8), and z neighbours are in-lane (row1 vs row0) or 8 lanes apart
//   (row0 vs the row1 of lane l-8).
// Partial (clipped) chunks use the same layout with invalid elements masked
// to zero, which is exactly the reference's "zero outside the chunk" rule
// (P/quantize.py:136-141, P/reconstruct.py:43-46).
#pragma once

#include "lzb_common.cuh"

namespace lzb {
namespace f3 {

constexpr uint32_t kFull = 0xffffffffu;

// ---------------------------------------------------------------------------
// prequantization (P/quantize.py:90-110)
// Fast path: q = x * (1/(2eb)) in f64; the integer is read off a magic-number
// add.  It is PROVABLY equal to the reference's trunc(RN(RN(x/2eb) +- 0.5))
// whenever |q| < 2^27 and q is at least 2^-16 away from a half-integer
// (|q - x/2eb| <= 2^-25 there), and then the reference's debug assert holds
// too.  Anything else takes the exact path.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int32_t pq_fast(double x, double inv, bool &ok) {
    const double M = 6755399441055744.0;  // 1.5 * 2^52
    double q = __dmul_rn(x, inv);
    double a = fabs(q);
    double t = __dadd_rn(a, M);
    double r = __dsub_rn(t, M);
    double f = __dsub_rn(a, r);
    ok = ok && (a < 134217728.0) && (fabs(f) < 0.4999847412109375);  // 2^27, 0.5 - 2^-16
    int32_t k = (int32_t)__double2loint(t);
    return q < 0.0 ? -k : k;
}

// f32-input fast path in FP32 arithmetic (2x the FP64 rate, no conversions):
// q = x * (inv_hi + inv_lo) with inv_hi + inv_lo = 1/(2eb) to ~2^-46.  The
// magic-number add is fused with the product, t = RN(x * inv_hi + M), so
// k = t - M is the integer nearest to the exact product x * inv_hi; the
// remainder against k is f = RN(x * inv_lo + RN(x * inv_hi - k)), within
// 2^-24 of x * inv - k for |k| < 2^22 (the inner FMA's argument is below 1/2
// in magnitude: rounding 2^-26; the outer sum below 1: 2^-25; the split of
// 1/(2eb): 2^-24).  Accepted only for |k| < 2^22 and |f| < 1/2 - 2^-16, where
// the error cannot change round-half-away(x / 2eb) nor the reference's debug
// assert; NaN inputs fail the remainder
// test, infinities both.  lzb_prequant_verify checks exactly this function
// against the exact rule over all 2^32 f32 bit patterns.
__device__ __forceinline__ int32_t pq_fast_f32(float x, float inv_hi, float inv_lo, bool &ok) {
    const float M = 12582912.0f;  // 1.5 * 2^23
    const float t = __fmaf_rn(x, inv_hi, M);
    const float k = __fsub_rn(t, M);
    const float f = __fmaf_rn(x, inv_lo, __fmaf_rn(x, inv_hi, -k));
    ok = ok && (fabsf(k) < 4194304.0f) && (fabsf(f) < 0.4999847412109375f);
    return __float_as_int(t) - 0x4B400000;  // integer value of k
}

// The same arithmetic for the K1 TMA path: the magnitude guard is folded
// into a running maximum `kmax` (the caller tests kmax < 2^22 once; NaN
// inputs still fail the remainder test), and the result is the BIASED
// integer float_as_int(t) = 0x4B400000 + k: the Lorenzo differences cancel
// the bias everywhere but at a chunk's origin element, which the caller
// corrects once (kPqBias).  Accepted exactly when pq_fast_f32 accepts.
constexpr int32_t kPqBias = 0x4B400000;
__device__ __forceinline__ int32_t pq_fast_f32b(float x, float inv_hi, float inv_lo, bool &ok, float &kmax) {
    const float M = 12582912.0f;
    const float t = __fmaf_rn(x, inv_hi, M);
    const float k = __fsub_rn(t, M);
    const float f = __fmaf_rn(x, inv_lo, __fmaf_rn(x, inv_hi, -k));
    ok = ok && (fabsf(f) < 0.4999847412109375f);
    kmax = fmaxf(kmax, fabsf(k));
    return __float_as_int(t);
}

// exact reference prequantization; flags: 1 overflow, 2 assert
__device__ __forceinline__ int64_t pq_exact(double v, double two_eb, double slack, int &flags) {
    double s = __ddiv_rn(v, two_eb);
    double r = trunc(__dadd_rn(s, copysign(0.5, s)));
    if (fabs(r) >= 576460752303423488.0) {
        flags |= 1;
        return 0;
    }
    int64_t c = (int64_t)r;
    double back = __dmul_rn((double)c, two_eb);
    if (!(fabs(__dsub_rn(v, back)) <= slack)) flags |= 2;
    return c;
}

// ---------------------------------------------------------------------------
// chunk geometry
// ---------------------------------------------------------------------------
struct Chunk {
    uint64_t x0, y0, z0;
    uint32_t ex, ey, ez;
    uint64_t base;  // chunk-major stream offset
    bool full;
};

__device__ __forceinline__ Chunk chunk_of(const Geom &g, uint64_t c) {
    Chunk k;
    uint64_t bx = c % g.nbx, t = c / g.nbx;
    uint64_t by = t % g.nby, bz = t / g.nby;
    k.x0 = bx * 8;
    k.y0 = by * 8;
    k.z0 = bz * 8;
    k.ex = (uint32_t)umin64(8, g.nx - k.x0);
    k.ey = (uint32_t)umin64(8, g.ny - k.y0);
    k.ez = (uint32_t)umin64(8, g.nz - k.z0);
    k.full = (k.ex == 8) & (k.ey == 8) & (k.ez == 8);
    k.base = g.nx * g.ny * 8 * bz + g.nx * (uint64_t)k.ez * 8 * by + (uint64_t)k.ez * k.ey * 8 * bx;
    return k;
}

// chunk at coordinates (bx, by, bz): no divisions
__device__ __forceinline__ Chunk chunk_at(const Geom &g, uint64_t bx, uint64_t by, uint64_t bz) {
    Chunk k;
    k.x0 = bx * 8;
    k.y0 = by * 8;
    k.z0 = bz * 8;
    k.ex = (uint32_t)umin64(8, g.nx - k.x0);
    k.ey = (uint32_t)umin64(8, g.ny - k.y0);
    k.ez = (uint32_t)umin64(8, g.nz - k.z0);
    k.full = (k.ex == 8) & (k.ey == 8) & (k.ez == 8);
    k.base = g.nx * g.ny * 8 * bz + g.nx * (uint64_t)k.ez * 8 * by + (uint64_t)k.ez * k.ey * 8 * bx;
    return k;
}

// next chunk ordinal: x-chunks fastest, then y, then z
__device__ __forceinline__ void chunk_step(const Geom &g, uint64_t &bx, uint64_t &by, uint64_t &bz) {
    if (++bx == g.nbx) {
        bx = 0;
        if (++by == g.nby) {
            by = 0;
            ++bz;
        }
    }
}

// local stream position of (lx, ly, lz) inside the chunk
__device__ __forceinline__ uint32_t lpos(const Chunk &k, uint32_t lx, uint32_t ly, uint32_t lz) {
    return lx + k.ex * (ly + k.ey * lz);
}

// ---------------------------------------------------------------------------
// Lorenzo deltas in registers (nested first differences, zero prepend)
// ---------------------------------------------------------------------------
// The lane masks are applied as multiply-adds by a 0/1 factor (one IMAD
// instead of a select + add per element and step).
template <typename I>
__device__ __forceinline__ void deltas(I (&v0)[8], I (&v1)[8], uint32_t lane) {
    const I fy = (lane & 7) ? I(1) : I(0);
    const I fz = lane >= 8 ? I(1) : I(0);
    // x
#pragma unroll
    for (int k = 7; k >= 1; k--) {
        v0[k] -= v0[k - 1];
        v1[k] -= v1[k - 1];
    }
    // y: previous row is lane - 1 inside the 8-lane group
#pragma unroll
    for (int k = 0; k < 8; k++) {
        I a = __shfl_up_sync(kFull, v0[k], 1, 8);
        I b = __shfl_up_sync(kFull, v1[k], 1, 8);
        v0[k] -= a * fy;
        v1[k] -= b * fy;
    }
    // z: row1 - row0 in lane; row0 - row1 of lane - 8
#pragma unroll
    for (int k = 0; k < 8; k++) {
        I up = __shfl_up_sync(kFull, v1[k], 8);
        v1[k] -= v0[k];
        v0[k] -= up * fz;
    }
}

// inclusive prefix sums along x, y, z (inverse of deltas)
template <typename I>
__device__ __forceinline__ void psums(I (&v0)[8], I (&v1)[8], uint32_t lane) {
    const uint32_t ly = lane & 7;
#pragma unroll
    for (int k = 1; k < 8; k++) {
        v0[k] += v0[k - 1];
        v1[k] += v1[k - 1];
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
        const I f = ly >= (uint32_t)o ? I(1) : I(0);
#pragma unroll
        for (int k = 0; k < 8; k++) {
            I a = __shfl_up_sync(kFull, v0[k], o, 8);
            I b = __shfl_up_sync(kFull, v1[k], o, 8);
            v0[k] += a * f;
            v1[k] += b * f;
        }
    }
    // z: pair (row0, row1) per lane, then across the four 8-lane groups
    const I f8 = lane >= 8 ? I(1) : I(0), f16 = lane >= 16 ? I(1) : I(0);
#pragma unroll
    for (int k = 0; k < 8; k++) {
        v1[k] += v0[k];
        I carry = v1[k];  // inclusive total of this lane's pair
        I s = carry;
        s += __shfl_up_sync(kFull, s, 8) * f8;
        s += __shfl_up_sync(kFull, s, 16) * f16;
        I excl = s - carry;
        v0[k] += excl;
        v1[k] += excl;
    }
}

// Rank of this lane's rows in chunk-major (stream) order, given per-row
// element counts c0 (row0) and c1 (row1).  Row order key = lz*8 + ly.
__device__ __forceinline__ void row_ranks(uint32_t c0, uint32_t c1, uint32_t lane, uint32_t &r0,
                                          uint32_t &r1, uint32_t &total) {
    uint32_t t = c0 + c1;
    uint32_t s = t;  // inclusive scan of t over the warp
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t a = __shfl_up_sync(kFull, s, o);
        if (lane >= (uint32_t)o) s += a;
    }
    total = __shfl_sync(kFull, s, 31);
    uint32_t gbase = __shfl_sync(kFull, s - t, lane & ~7u);  // sum of groups before
    uint32_t a0 = c0, a1 = c1;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
        uint32_t x = __shfl_up_sync(kFull, a0, o, 8);
        uint32_t y = __shfl_up_sync(kFull, a1, o, 8);
        if ((lane & 7) >= (uint32_t)o) {
            a0 += x;
            a1 += y;
        }
    }
    uint32_t g0 = __shfl_sync(kFull, a0, (lane & ~7u) | 7u);  // group total of row0 counts
    r0 = gbase + a0 - c0;
    r1 = gbase + g0 + a1 - c1;
}

}  // namespace f3
}  // namespace lzb
