// K6 fast path for ChunkSpec(8,8,8): one warp per chunk, eight consecutive
// chunk ordinals per warp task.  Included by lzb_recon.cu.  Semantics as the
// generic K6 (P/reconstruct.py:22-88, P/pipeline.py:108-117); register layout
// in lzb_fast3d.cuh.
//
// Per chunk: the lane's two 8-symbol rows are one 16-byte load each (the
// chunk is 1 KB contiguous in the chunk-major stream), q' = code - r, the
// chunk's outliers (bucketed per warp tile by a counting sort) are added, then
// inclusive scans along x (in registers), y (3 shuffle steps inside 8-lane
// groups) and z (in-lane pair + 2 shuffle steps), and the f64 dequantisation
// feeds two 32-byte row stores in grid order plus a running min/max.
// Values that might leave int32 (an outlier |delta| >= 2^20) send the chunk
// to the exact int64 variant with the reference's f64 prefix-sum guard.
#pragma once

#include "lzb_fast3d.cuh"

namespace lzb {

constexpr int kR3Warps = 8;
constexpr int kR3Threads = kR3Warps * 32;
constexpr int kR3TileChunks = 8;

struct R3Params {
    const void *codes;
    Geom g;
    double two_eb;
    int32_t r;
    void *y;
    int64_t *pre;             // optional int64 prequant output
    lzb_dstatus *st;
    unsigned long long *mm;   // [min key, max key, first bad offset]
    uint64_t nchunks, ntiles;
    const uint64_t *tile_start;  // ntiles + 1
    const uint64_t *brec;        // per record: [k << 9 | lz << 6 | ly << 3 | lx, delta]
    unsigned int *ticket;
    int vec_ok;
    int codes_vec;  // the code stream is 16-byte aligned: vector / cp.async loads of full chunks
};

__device__ __forceinline__ unsigned long long r3_dkey(double v) {
    unsigned long long b = __double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

template <typename I>
__device__ __forceinline__ void r3_add_outliers(const R3Params &p, uint64_t r0, uint64_t r1,
                                                uint32_t k, uint32_t lane, I (&v0)[8], I (&v1)[8]) {
    const uint32_t ly = lane & 7, lz0 = (lane >> 3) * 2;
    for (uint64_t i = r0; i < r1; i++) {
        const uint64_t key = p.brec[2 * i];
        if ((uint32_t)(key >> 9) != k) continue;
        const int64_t d = (int64_t)p.brec[2 * i + 1];
        const uint32_t lx = key & 7, oy = (key >> 3) & 7, oz = (key >> 6) & 7;
        if (oy != ly) continue;
        if (oz == lz0) {
#pragma unroll
            for (int j = 0; j < 8; j++)
                if ((uint32_t)j == lx) v0[j] += (I)d;
        } else if (oz == lz0 + 1) {
#pragma unroll
            for (int j = 0; j < 8; j++)
                if ((uint32_t)j == lx) v1[j] += (I)d;
        }
    }
}

// does any record of chunk k carry a delta too large for the int32 path?
__device__ __forceinline__ bool r3_needs_wide(const R3Params &p, uint64_t r0, uint64_t r1, uint32_t k) {
    bool wide = false;
    for (uint64_t i = r0 + lane_id(); i < r1; i += 32) {
        const uint64_t key = p.brec[2 * i];
        const int64_t d = (int64_t)p.brec[2 * i + 1];
        if ((uint32_t)(key >> 9) == k && (d >= (1ll << 20) || d <= -(1ll << 20))) wide = true;
    }
    return __any_sync(f3::kFull, wide);
}

// The tile's outliers held in registers (lane i: record i, i < 32): apply
// those of chunk k.  Usually at most the chunk origin.
template <typename I>
__device__ __forceinline__ void r3_add_reg(uint32_t rkey, int32_t rd, uint32_t nrec, uint32_t k,
                                           uint32_t lane, I (&v0)[8], I (&v1)[8]) {
    uint32_t m = __ballot_sync(f3::kFull, lane < nrec && (rkey >> 9) == k);
    const uint32_t ly = lane & 7, lz0 = (lane >> 3) * 2;
    while (m) {
        const uint32_t i = __ffs(m) - 1;
        m &= m - 1;
        const uint32_t key = __shfl_sync(f3::kFull, rkey, i);
        const int32_t d = __shfl_sync(f3::kFull, rd, i);
        const uint32_t lx = key & 7, oy = (key >> 3) & 7, oz = (key >> 6) & 7;
        const bool mine = oy == ly && (oz & ~1u) == lz0;
        const bool r1 = oz & 1u;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const I add = (mine && (uint32_t)j == lx) ? (I)d : (I)0;
            v0[j] += r1 ? (I)0 : add;
            v1[j] += r1 ? add : (I)0;
        }
    }
}

// ---------------------------------------------------------------------------
// Packed 16-bit reconstruction (cap <= 4096).  All partial sums are taken
// modulo 2^16, two x-neighbours per register (VIADD.16x2); the results are
// exact whenever every partial sum of the chunk fits int16, which holds when
// sum |q'| over the chunk < 2^15 -- checked first, exactly (codes give |q'| <
// 2048, at most 8 per 16-bit half, so the packed sum of |q'| cannot wrap).
// Chunks that fail the check take the int32 path.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t v2add(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("add.s16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
__device__ __forceinline__ uint32_t v2min(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("min.s16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
__device__ __forceinline__ uint32_t v2max(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("max.s16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
// v += (value of lane - o inside the 2^k-lane segment given by c), if that lane exists
__device__ __forceinline__ void v2_shfl_add(uint32_t &v, uint32_t src, uint32_t o, uint32_t c) {
    asm volatile("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
        "shfl.sync.up.b32 t|p, %1, %2, %3, -1;\n\t"
        "@p add.s16x2 %0, %0, t;\n\t}"
        : "+r"(v)
        : "r"(src), "r"(o), "r"(c));
}
__device__ __forceinline__ int32_t v2lo(uint32_t v) { return (int32_t)(v << 16) >> 16; }
__device__ __forceinline__ int32_t v2hi(uint32_t v) { return (int32_t)v >> 16; }

// Returns false (nothing written) when the chunk is not provably exact in 16 bits.
// qa / qb: the lane's two code rows (ly, lz0) and (ly, lz0 + 1).
__device__ __forceinline__ bool r3_chunk16(const R3Params &p, const uint4 qa, const uint4 qb, uint32_t k,
                                          uint32_t lane, uint32_t &mn, uint32_t &mx, uint32_t rkey, int32_t rd,
                                          uint32_t nrec, uint32_t ybuf_s) {
    const uint32_t ly = lane & 7, lz0 = (lane >> 3) * 2;
    const uint32_t nr = ((uint32_t)(-p.r) & 0xFFFFu) * 0x10001u;  // -r in both halves
    uint32_t a[4] = {v2add(qa.x, nr), v2add(qa.y, nr), v2add(qa.z, nr), v2add(qa.w, nr)};
    uint32_t b[4] = {v2add(qb.x, nr), v2add(qb.y, nr), v2add(qb.z, nr), v2add(qb.w, nr)};
    // exactness: sum |q'| over the chunk (codes, then the outlier deltas) < 2^15
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        acc = v2add(acc, v2max(a[i], v2add(~a[i], 0x00010001u)));
        acc = v2add(acc, v2max(b[i], v2add(~b[i], 0x00010001u)));
    }
    const bool mine_rec = lane < nrec && (rkey >> 9) == k;
    const uint32_t dabs = mine_rec ? (uint32_t)min(abs(rd), 0x8000) : 0u;
    const uint32_t S = __reduce_add_sync(f3::kFull, (acc & 0xFFFFu) + (acc >> 16) + dabs);
    if (S >= 0x8000u) return false;
    // outliers: q'[idx] += delta (mod 2^16 in its half)
    for (uint32_t m = __ballot_sync(f3::kFull, mine_rec); m; m &= m - 1) {
        const uint32_t i = __ffs(m) - 1;
        const uint32_t key = __shfl_sync(f3::kFull, rkey, i);
        const uint32_t d16 = (uint32_t)__shfl_sync(f3::kFull, rd, i) & 0xFFFFu;
        const uint32_t lx = key & 7, oy = (key >> 3) & 7, oz = (key >> 6) & 7;
        const bool own = oy == ly && (oz & ~1u) == lz0;
        const uint32_t add = own ? (d16 << (16 * (lx & 1))) : 0u;
        const uint32_t w = lx >> 1;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const uint32_t aj = (j == (int)w && !(oz & 1)) ? add : 0u, bj = (j == (int)w && (oz & 1)) ? add : 0u;
            a[j] = v2add(a[j], aj);
            b[j] = v2add(b[j], bj);
        }
    }
    // x: inside each pair, then the running pair totals
#pragma unroll
    for (int i = 0; i < 4; i++) {
        a[i] = v2add(a[i], a[i] << 16);
        b[i] = v2add(b[i], b[i] << 16);
    }
#pragma unroll
    for (int i = 1; i < 4; i++) {
        a[i] = v2add(a[i], __byte_perm(a[i - 1], 0, 0x3232));
        b[i] = v2add(b[i], __byte_perm(b[i - 1], 0, 0x3232));
    }
    // y: previous rows in the 8-lane group
#pragma unroll
    for (uint32_t o = 1; o < 8; o <<= 1) {
#pragma unroll
        for (int i = 0; i < 4; i++) {
            v2_shfl_add(a[i], a[i], o, 0x1800u);
            v2_shfl_add(b[i], b[i], o, 0x1800u);
        }
    }
    // z: the lane's pair, then the groups of 8 lanes below
#pragma unroll
    for (int i = 0; i < 4; i++) {
        b[i] = v2add(b[i], a[i]);
        uint32_t e = 0;
        v2_shfl_add(e, b[i], 8, 0u);
        const uint32_t s2 = v2add(e, b[i]);
        v2_shfl_add(e, s2, 16, 0u);
        a[i] = v2add(a[i], e);
        b[i] = v2add(b[i], e);
        mn = v2min(mn, v2min(a[i], b[i]));
        mx = v2max(mx, v2max(a[i], b[i]));
    }
    // dequantise (f64 multiply, RN to f32) into the TMA tile
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const uint32_t(&v)[4] = h ? b : a;
        float o[8];
#pragma unroll
        for (int i = 0; i < 4; i++) {
            o[2 * i] = (float)__dmul_rn((double)v2lo(v[i]), p.two_eb);
            o[2 * i + 1] = (float)__dmul_rn((double)v2hi(v[i]), p.two_eb);
        }
        const uint32_t sa = ybuf_s + (ly + 8 * (lz0 + h)) * 32;
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(sa), "f"(o[0]), "f"(o[1]), "f"(o[2]),
                     "f"(o[3]));
        asm volatile("st.shared.v4.f32 [%0+16], {%1, %2, %3, %4};" ::"r"(sa), "f"(o[4]), "f"(o[5]), "f"(o[6]),
                     "f"(o[7]));
    }
    return true;
}

template <typename SymT, typename OutT, typename I>
__device__ __forceinline__ void r3_chunk(const R3Params &p, const f3::Chunk &ch, uint32_t k,
                                         uint64_t r0, uint64_t r1, uint32_t lane, OutT &vmin,
                                         OutT &vmax, bool &overflow, const SymT *stg = nullptr,
                                         bool reg_out = false, uint32_t rkey = 0, int32_t rd = 0,
                                         uint32_t nrec = 0, uint32_t ybuf_s = 0) {
    const uint32_t ly = lane & 7, lz0 = (lane >> 3) * 2;
    const SymT *cs = static_cast<const SymT *>(p.codes) + ch.base;
    I v0[8], v1[8];
    const uint32_t xmask = (1u << ch.ex) - 1u;
    const uint32_t m0 = (ly < ch.ey && lz0 < ch.ez) ? xmask : 0u;
    const uint32_t m1 = (ly < ch.ey && lz0 + 1 < ch.ez) ? xmask : 0u;
    const bool fast = ch.full && ((ch.base & 7) == 0) && p.codes_vec;
    if (fast) {
#pragma unroll
        for (int h = 0; h < 2; h++) {
            I(&v)[8] = h ? v1 : v0;
            const SymT *src = cs + 8 * (ly + 8 * (lz0 + h));
            if constexpr (sizeof(SymT) == 2) {
                uint4 a = stg ? reinterpret_cast<const uint4 *>(stg)[32 * h]
                              : __ldg(reinterpret_cast<const uint4 *>(src));
                uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    v[2 * j] = (I)(int32_t)(w[j] & 0xFFFFu) - p.r;
                    v[2 * j + 1] = (I)(int32_t)(w[j] >> 16) - p.r;
                }
            } else {
                uint4 a, b;
                if (stg) {
                    a = reinterpret_cast<const uint4 *>(stg)[32 * (2 * h)];
                    b = reinterpret_cast<const uint4 *>(stg)[32 * (2 * h + 1)];
                } else {
                    a = __ldg(reinterpret_cast<const uint4 *>(src));
                    b = __ldg(reinterpret_cast<const uint4 *>(src) + 1);
                }
                uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
                for (int j = 0; j < 8; j++) v[j] = (I)(int64_t)w[j] - p.r;
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < 8; j++) {
            v0[j] = ((m0 >> j) & 1u) ? (I)(int64_t)cs[f3::lpos(ch, j, ly, lz0)] - p.r : (I)0;
            v1[j] = ((m1 >> j) & 1u) ? (I)(int64_t)cs[f3::lpos(ch, j, ly, lz0 + 1)] - p.r : (I)0;
        }
    }
    if (reg_out) r3_add_reg<I>(rkey, rd, nrec, k, lane, v0, v1);
    else if (r1 > r0) r3_add_outliers<I>(p, r0, r1, k, lane, v0, v1);
    if constexpr (sizeof(I) == 8) {
        // prefix-sum magnitude guard (P/reconstruct.py:48-53), f64 sum per chunk
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < 8; j++) s += fabs((double)v0[j]) + fabs((double)v1[j]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(f3::kFull, s, o);
        if (s >= 4611686018427387904.0) overflow = true;
    }
    f3::psums<I>(v0, v1, lane);
    OutT *yo = static_cast<OutT *>(p.y);
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const I(&v)[8] = h ? v1 : v0;
        const uint32_t mm = h ? m1 : m0;
        OutT o[8];
#pragma unroll
        for (int j = 0; j < 8; j++) o[j] = (OutT)__dmul_rn((double)v[j], p.two_eb);
        if (fast) {  // outputs are never NaN: plain min/max instructions
#pragma unroll
            for (int j = 0; j < 8; j++) {
                vmin = fmin(vmin, o[j]);
                vmax = fmax(vmax, o[j]);
            }
        } else {
#pragma unroll
            for (int j = 0; j < 8; j++)
                if ((mm >> j) & 1u) {
                    vmin = fmin(vmin, o[j]);
                    vmax = fmax(vmax, o[j]);
                }
        }
        if (fast && ybuf_s) {  // into the warp's TMA store tile: row ly + 8 lz, 32 bytes
            if constexpr (sizeof(OutT) == 4) {
                const uint32_t a = ybuf_s + (ly + 8 * (lz0 + h)) * 32;
                asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(o[0]), "f"(o[1]), "f"(o[2]),
                             "f"(o[3]));
                asm volatile("st.shared.v4.f32 [%0+16], {%1, %2, %3, %4};" ::"r"(a), "f"(o[4]), "f"(o[5]),
                             "f"(o[6]), "f"(o[7]));
            }
        } else if (fast && p.vec_ok) {
            const uint64_t gi = ch.x0 + p.g.nx * ((ch.y0 + ly) + p.g.ny * (ch.z0 + lz0 + h));
            if constexpr (sizeof(OutT) == 4) {
                float4 *dst = reinterpret_cast<float4 *>(yo + gi);
                dst[0] = make_float4(o[0], o[1], o[2], o[3]);
                dst[1] = make_float4(o[4], o[5], o[6], o[7]);
            } else {
                double2 *dst = reinterpret_cast<double2 *>(yo + gi);
#pragma unroll
                for (int j = 0; j < 4; j++) dst[j] = make_double2(o[2 * j], o[2 * j + 1]);
            }
            if (p.pre)
#pragma unroll
                for (int j = 0; j < 8; j++) p.pre[gi + j] = (int64_t)v[j];
        } else if (mm) {
            const uint64_t gi = ch.x0 + p.g.nx * ((ch.y0 + ly) + p.g.ny * (ch.z0 + lz0 + h));
#pragma unroll
            for (int j = 0; j < 8; j++)
                if ((mm >> j) & 1u) {
                    yo[gi + j] = o[j];
                    if (p.pre) p.pre[gi + j] = (int64_t)v[j];
                }
        }
    }
}

template <typename SymT, typename OutT>
__device__ __noinline__ void r3_chunk_wide(const R3Params *pp, uint64_t c, uint32_t k, uint64_t r0,
                                           uint64_t r1, uint32_t lane, OutT *mm, bool *ovf) {
    const f3::Chunk ch = f3::chunk_of(pp->g, c);
    OutT vmin = mm[0], vmax = mm[1];
    bool o = *ovf;
    r3_chunk<SymT, OutT, int64_t>(*pp, ch, k, r0, r1, lane, vmin, vmax, o);
    mm[0] = vmin;
    mm[1] = vmax;
    *ovf = o;
}

// the lane's two code rows of a full chunk -> its stage slot (cp.async)
template <typename SymT>
__device__ __forceinline__ void r3_prefetch(const R3Params &p, const f3::Chunk &ch, uint32_t lane,
                                            uint32_t saddr) {
    const SymT *cs = static_cast<const SymT *>(p.codes) + ch.base;
    const uint32_t ly = lane & 7, lz0 = (lane >> 3) * 2;
    constexpr int V = 16 / sizeof(SymT);  // symbols per 16-byte copy
#pragma unroll
    for (int h = 0; h < 2; h++)
#pragma unroll
        for (int k = 0; k < 8 / V; k++)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr + 512 * (h * (8 / V) + k)),
                         "l"(cs + 8 * (ly + 8 * (lz0 + h)) + V * k)
                         : "memory");
}

// TMA store of one finished chunk (8x8x8 f32 box) from the warp's tile buffer
__device__ __forceinline__ void r3_tma_store(const CUtensorMap *map, uint32_t src, uint64_t x, uint64_t y,
                                             uint64_t z) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"((int)x), "r"((int)y), "r"((int)z), "r"(src)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// TMA: full f32 chunks leave through a per-warp double-buffered shared tile
// and one TMA tensor store each (the 32-byte row fragments of a chunk are
// scattered over 64 rows; as plain stores they saturate L1).
template <typename SymT, typename OutT, bool TMA>
__global__ void __launch_bounds__(kR3Threads, TMA ? 3 : 3)
    k_reconstruct3d8(const __grid_constant__ R3Params p, const __grid_constant__ CUtensorMap ymap) {
    // per-warp double buffer of the next chunk's code rows (16 symbols per lane)
    __shared__ __align__(16) SymT s_stage[kR3Warps][2][32 * 16];
    // TMA: per-warp double-buffered 2 KB output tiles (dynamic shared memory)
    extern __shared__ __align__(128) float s_y[];
    const uint32_t ybase_s = (uint32_t)__cvta_generic_to_shared(s_y) + (threadIdx.x >> 5) * 4096;
    uint32_t nb = 0;  // TMA store tiles issued by this warp
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    // piece-major: 16-byte piece k of lane l at byte k * 512 + 16 l (conflict-free)
    const uint32_t stage_s = (uint32_t)__cvta_generic_to_shared(&s_stage[warp][0][0]) + lane * 16;
    constexpr uint32_t kBuf = 32 * 16 * sizeof(SymT);
    OutT vmin = (OutT)INFINITY, vmax = (OutT)-INFINITY;
    uint32_t qmn = 0x7FFF7FFFu, qmx = 0x80008000u;  // packed int16 min / max of the 16-bit path's q
    const bool narrow = p.r <= 2048;                 // cap <= 4096
    bool overflow = false;
    while (true) {
        uint64_t t = 0;
        if (lane == 0) t = atomicAdd(p.ticket, 1u);
        t = __shfl_sync(f3::kFull, t, 0);
        if (t >= p.ntiles) break;
        t = p.ntiles - 1 - t;  // tiles from the end first (partial chunks; see k_quantize3d8)
        const uint64_t c0 = t * kR3TileChunks;
        const uint64_t c1 = umin64(c0 + kR3TileChunks, p.nchunks);
        const uint64_t r0 = p.tile_start[t], r1 = p.tile_start[t + 1];
        // outliers of the tile: up to 32 in registers (one per lane), with a
        // per-chunk mask of chunks that need the exact int64 path
        const uint64_t nr64 = r1 - r0;
        const bool reg_out = nr64 <= 32;
        const uint32_t nrec = reg_out ? (uint32_t)nr64 : 0u;
        uint32_t rkey = 0xFFFFFFFFu;
        int32_t rd = 0;
        uint32_t wide_mask = 0;
        if (reg_out) {
            bool wide = false;
            if (lane < nrec) {
                rkey = (uint32_t)p.brec[2 * (r0 + lane)];
                const int64_t d = (int64_t)p.brec[2 * (r0 + lane) + 1];
                wide = d >= (1ll << 20) || d <= -(1ll << 20);
                rd = (int32_t)d;
            }
            const uint32_t wm = __ballot_sync(f3::kFull, wide);
            for (uint32_t m = wm; m; m &= m - 1)
                wide_mask |= 1u << (__shfl_sync(f3::kFull, rkey, __ffs(m) - 1) >> 9);
        }
        uint64_t cbx = c0 % p.g.nbx, cby = (c0 / p.g.nbx) % p.g.nby, cbz = (c0 / p.g.nbx) / p.g.nby;
        f3::Chunk cur = f3::chunk_at(p.g, cbx, cby, cbz);
        bool cur_pf = cur.full && (cur.base & 7) == 0 && p.codes_vec;
        if (cur_pf) r3_prefetch<SymT>(p, cur, lane, stage_s);
        asm volatile("cp.async.commit_group;" ::: "memory");
        uint32_t sb = 0;
        for (uint64_t c = c0; c < c1; c++) {
            const uint32_t k = (uint32_t)(c - c0);
            f3::Chunk nxt;
            bool nxt_pf = false;
            if (c + 1 < c1) {
                if (cbx + 1 < p.g.nbx) {  // same chunk row: advance along x
                    cbx++;
                    nxt = cur;
                    nxt.x0 += 8;
                    nxt.base += (uint64_t)cur.ez * cur.ey * 8;
                    nxt.ex = (uint32_t)umin64(8, p.g.nx - nxt.x0);
                    nxt.full = (nxt.ex == 8) & (nxt.ey == 8) & (nxt.ez == 8);
                } else {
                    f3::chunk_step(p.g, cbx, cby, cbz);
                    nxt = f3::chunk_at(p.g, cbx, cby, cbz);
                }
                nxt_pf = nxt.full && (nxt.base & 7) == 0 && p.codes_vec;
                if (nxt_pf) r3_prefetch<SymT>(p, nxt, lane, stage_s + (sb ^ 1) * kBuf);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            asm volatile("cp.async.wait_group 1;" ::: "memory");
            // warp-uniform by construction; the vote tells the compiler so,
            // which keeps the chunk's shuffles free of divergence handling
            const bool wide = __any_sync(f3::kFull, reg_out ? ((wide_mask >> k) & 1u) != 0
                                                            : (r1 > r0 && r3_needs_wide(p, r0, r1, k)));
            if (wide) {
                OutT mmv[2] = {vmin, vmax};
                r3_chunk_wide<SymT, OutT>(&p, c, k, r0, r1, lane, mmv, &overflow);
                vmin = mmv[0];
                vmax = mmv[1];
            } else {
                const bool tma = TMA && p.codes_vec && __any_sync(f3::kFull, cur.full);  // = r3_chunk's fast
                uint32_t yb = 0;
                if (tma) {
                    yb = ybase_s + (nb & 1u) * 2048;
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                    __syncwarp();
                }
                const SymT *stg = cur_pf ? reinterpret_cast<const SymT *>(
                                               reinterpret_cast<const unsigned char *>(&s_stage[warp][sb][0]) + lane * 16)
                                         : nullptr;
                bool done = false;
                if constexpr (sizeof(SymT) == 2 && sizeof(OutT) == 4 && TMA) {
                    // packed 16-bit partial sums when provably exact (cap <= 4096)
                    if (narrow && reg_out && __all_sync(f3::kFull, cur_pf))
                        done = r3_chunk16(p, reinterpret_cast<const uint4 *>(stg)[0],
                                          reinterpret_cast<const uint4 *>(stg)[32], k, lane, qmn, qmx, rkey, rd, nrec,
                                          yb);
                }
                if (!done)
                    r3_chunk<SymT, OutT, int32_t>(p, cur, k, r0, r1, lane, vmin, vmax, overflow, stg, reg_out, rkey,
                                                  rd, nrec, yb);
                if (tma) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) r3_tma_store(&ymap, yb, cur.x0, cur.y0, cur.z0);
                    nb++;
                }
            }
            cur = nxt;
            cur_pf = nxt_pf;
            sb ^= 1;
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    if (TMA && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    {  // the 16-bit path's extremes: the dequantisation is monotone in q
        const int32_t lo = min(v2lo(qmn), v2hi(qmn)), hi = max(v2lo(qmx), v2hi(qmx));
        if (lo <= hi) {
            vmin = fmin(vmin, (OutT)__dmul_rn((double)lo, p.two_eb));
            vmax = fmax(vmax, (OutT)__dmul_rn((double)hi, p.two_eb));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        OutT a = __shfl_xor_sync(f3::kFull, vmin, o), b = __shfl_xor_sync(f3::kFull, vmax, o);
        vmin = fmin(vmin, a);
        vmax = fmax(vmax, b);
    }
    if (lane == 0 && vmin <= vmax) {
        atomicMin(&p.mm[0], r3_dkey((double)vmin));
        atomicMax(&p.mm[1], r3_dkey((double)vmax));
    }
    if (__any_sync(f3::kFull, overflow) && lane == 0) set_status(p.st, LZB_E_OVERFLOW);
}

// Non-finite outputs are rare (an overflowing dequantisation).  The running
// min/max already see any +-inf; only then does this pass look for the first
// offending offset (the reference reports it, P/grid.py:176-180).
template <typename OutT>
__global__ void k_first_nonfinite(const OutT *y, uint64_t n, unsigned long long *mm) {
    const unsigned long long kinf_lo = r3_dkey(-INFINITY), kinf_hi = r3_dkey(INFINITY);
    if (mm[0] != kinf_lo && mm[1] != kinf_hi) return;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        if (!isfinite((double)y[i])) atomicMin(&mm[2], (unsigned long long)i);
}

}  // namespace lzb
