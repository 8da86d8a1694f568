// K6 for 2D fields with ChunkSpec(16,16) and 1D fields with ChunkSpec(256):
// one warp per 256-element chunk, eight consecutive chunk ordinals per warp
// task.  Included by lzb_recon.cu.
// Semantics as the generic K6 (P/reconstruct.py:22-88, P/pipeline.py:108-117).
//
// Register layout as K1's (lzb_quant2d.cuh): lane l owns the chunk stream
// positions 8 l .. 8 l + 7 (2D: row l >> 1, x = 8 (l & 1) ..; 1D: x = 8 l ..),
// so its eight codes are one 16-byte load from the chunk-major stream; an
// outlier record's key is k << 8 | (chunk stream position).  q' = code - r,
// the chunk's outliers (bucketed per warp tile, up to 32 held one per lane)
// are added, then the inverse Lorenzo: an inclusive scan along x (in-lane,
// plus the lanes to the left: one shuffle in 2D, a five-step warp scan in
// 1D) and in 2D along y (rows are lanes two apart: four shuffle steps), and
// the f64 dequantisation feeds two 16-byte row stores.  int32 partial sums
// are exact while every outlier |delta| < 2^20 (|sum| < 256 * (2^15 + 2^20)
// < 2^29); other chunks take the int64 variant with the reference's f64
// prefix-sum guard (P/reconstruct.py:48-53).
#pragma once

#include "lzb_recon3d.cuh"

namespace lzb {

struct R2Chunk {
    uint64_t x0, y0, base;
    uint32_t ex, ey;
    bool full;
};

template <int D>
__device__ __forceinline__ R2Chunk r2_chunk_of(const Geom &g, uint64_t c) {
    R2Chunk k;
    if constexpr (D == 1) {
        k.x0 = c * 256;
        k.y0 = 0;
        k.ex = (uint32_t)umin64(256, g.nx - k.x0);
        k.ey = 1;
        k.full = k.ex == 256;
        k.base = k.x0;
    } else {
        const uint64_t by = c / g.nbx, bx = c - by * g.nbx;
        k.x0 = bx * 16;
        k.y0 = by * 16;
        k.ex = (uint32_t)umin64(16, g.nx - k.x0);
        k.ey = (uint32_t)umin64(16, g.ny - k.y0);
        k.full = k.ex == 16 && k.ey == 16;
        k.base = g.nx * 16 * by + (uint64_t)k.ey * 16 * bx;
    }
    return k;
}

template <int D>
__device__ __forceinline__ uint32_t r2_vmask(const R2Chunk &k, uint32_t lane) {
    const uint32_t xh = D == 1 ? 8 * lane : 8 * (lane & 1), ly = D == 1 ? 0u : lane >> 1;
    if (ly >= k.ey || xh >= k.ex) return 0u;
    const uint32_t w = k.ex - xh;
    return w >= 8 ? 0xFFu : ((1u << w) - 1u);
}

template <int D>
__device__ __forceinline__ uint64_t r2_lane_gi(const R2Chunk &k, uint32_t lane, uint64_t nx) {
    if constexpr (D == 1) return k.x0 + 8 * lane;
    else return (k.x0 + 8 * (lane & 1)) + nx * (k.y0 + (lane >> 1));
}

// the lane's eight codes (raw, not yet centred); 16-byte load for full chunks
template <int D, typename SymT>
__device__ __forceinline__ void r2_load(const R3Params &p, const R2Chunk &k, uint32_t lane, uint32_t vm,
                                        uint32_t (&c)[8]) {
    const SymT *cs = static_cast<const SymT *>(p.codes) + k.base;
    if (k.full && p.codes_vec) {
        if constexpr (sizeof(SymT) == 2) {
            const uint4 a = __ldg(reinterpret_cast<const uint4 *>(cs + 8 * lane));
            const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
            for (int j = 0; j < 4; j++) {
                c[2 * j] = w[j] & 0xFFFFu;
                c[2 * j + 1] = w[j] >> 16;
            }
        } else {
            const uint4 a = __ldg(reinterpret_cast<const uint4 *>(cs + 8 * lane));
            const uint4 b = __ldg(reinterpret_cast<const uint4 *>(cs + 8 * lane) + 1);
            c[0] = a.x; c[1] = a.y; c[2] = a.z; c[3] = a.w;
            c[4] = b.x; c[5] = b.y; c[6] = b.z; c[7] = b.w;
        }
    } else {
        const uint32_t pos0 = D == 1 ? 8 * lane : (lane >> 1) * k.ex + 8 * (lane & 1);  // full: 8 lane
#pragma unroll
        for (int j = 0; j < 8; j++) c[j] = ((vm >> j) & 1u) ? (uint32_t)cs[pos0 + j] : 0u;
    }
}

// records of the tile's chunk k: key = k << 8 | chunk stream position (8 lane + j)
template <typename I>
__device__ __forceinline__ void r2_add_reg(uint32_t rkey, int64_t rd, uint32_t nrec, uint32_t k, uint32_t lane,
                                           I (&v)[8]) {
    uint32_t m = __ballot_sync(f3::kFull, lane < nrec && (rkey >> 8) == k);
    while (m) {
        const uint32_t i = __ffs(m) - 1;
        m &= m - 1;
        const uint32_t key = __shfl_sync(f3::kFull, rkey, i);
        const int64_t d = __shfl_sync(f3::kFull, rd, i);
        const bool mine = ((key & 255u) >> 3) == lane;
#pragma unroll
        for (int j = 0; j < 8; j++)
            if (mine && (uint32_t)j == (key & 7u)) v[j] += (I)d;
    }
}

template <typename I>
__device__ __forceinline__ void r2_add_list(const R3Params &p, uint64_t r0, uint64_t r1, uint32_t k, uint32_t lane,
                                            I (&v)[8]) {
    for (uint64_t i = r0; i < r1; i++) {
        const uint32_t key = (uint32_t)p.brec[2 * i];
        if ((key >> 8) != k || ((key & 255u) >> 3) != lane) continue;
        const int64_t d = (int64_t)p.brec[2 * i + 1];
#pragma unroll
        for (int j = 0; j < 8; j++)
            if ((uint32_t)j == (key & 7u)) v[j] += (I)d;
    }
}

// inverse Lorenzo: inclusive prefix sums along x (then y in 2D)
template <int D, typename I>
__device__ __forceinline__ void r2_psums(I (&v)[8], uint32_t lane) {
#pragma unroll
    for (int j = 1; j < 8; j++) v[j] += v[j - 1];
    if constexpr (D == 1) {  // exclusive warp scan of the lane totals
        I run = v[7];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const I a = __shfl_up_sync(f3::kFull, run, o);
            if (lane >= (uint32_t)o) run += a;
        }
        const I before = run - v[7];
#pragma unroll
        for (int j = 0; j < 8; j++) v[j] += before;
    } else {
        const I left = __shfl_up_sync(f3::kFull, v[7], 1);
        if (lane & 1) {
#pragma unroll
            for (int j = 0; j < 8; j++) v[j] += left;
        }
#pragma unroll
        for (int o = 2; o < 32; o <<= 1) {
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const I a = __shfl_up_sync(f3::kFull, v[j], o);
                if (lane >= (uint32_t)o) v[j] += a;
            }
        }
    }
}

template <int D, typename SymT, typename OutT, typename I>
__device__ __forceinline__ void r2_chunk(const R3Params &p, const R2Chunk &ch, const uint32_t (&c)[8], uint32_t k,
                                         uint64_t r0, uint64_t r1, bool reg_out, uint32_t rkey, int64_t rd,
                                         uint32_t nrec, uint32_t lane, OutT &vmin, OutT &vmax, bool &overflow) {
    const uint32_t vm = r2_vmask<D>(ch, lane);
    I v[8];
#pragma unroll
    for (int j = 0; j < 8; j++) v[j] = ((vm >> j) & 1u) ? (I)(int64_t)c[j] - (I)p.r : (I)0;
    if (reg_out) r2_add_reg<I>(rkey, rd, nrec, k, lane, v);
    else if (r1 > r0) r2_add_list<I>(p, r0, r1, k, lane, v);
    if constexpr (sizeof(I) == 8) {  // f64 prefix-sum guard per chunk
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < 8; j++) s += fabs((double)v[j]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(f3::kFull, s, o);
        if (s >= 4611686018427387904.0) overflow = true;
    }
    r2_psums<D, I>(v, lane);
    OutT o[8];
#pragma unroll
    for (int j = 0; j < 8; j++) o[j] = (OutT)__dmul_rn((double)v[j], p.two_eb);
    OutT *yo = static_cast<OutT *>(p.y);
    const uint64_t gi = r2_lane_gi<D>(ch, lane, p.g.nx);
    if (ch.full) {
#pragma unroll
        for (int j = 0; j < 8; j++) {
            vmin = fmin(vmin, o[j]);
            vmax = fmax(vmax, o[j]);
        }
    } else {
#pragma unroll
        for (int j = 0; j < 8; j++)
            if ((vm >> j) & 1u) {
                vmin = fmin(vmin, o[j]);
                vmax = fmax(vmax, o[j]);
            }
    }
    if (ch.full && p.vec_ok) {
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
    } else {
#pragma unroll
        for (int j = 0; j < 8; j++)
            if ((vm >> j) & 1u) {
                yo[gi + j] = o[j];
                if (p.pre) p.pre[gi + j] = (int64_t)v[j];
            }
    }
}

template <int D, typename SymT, typename OutT>
__device__ __noinline__ void r2_chunk_wide(const R3Params *pp, uint64_t c, uint32_t k, uint64_t r0, uint64_t r1,
                                           uint32_t lane, OutT *mm, bool *ovf) {
    const R2Chunk ch = r2_chunk_of<D>(pp->g, c);
    uint32_t cc[8];
    r2_load<D, SymT>(*pp, ch, lane, r2_vmask<D>(ch, lane), cc);
    OutT vmin = mm[0], vmax = mm[1];
    bool o = *ovf;
    r2_chunk<D, SymT, OutT, int64_t>(*pp, ch, cc, k, r0, r1, false, 0, 0, 0, lane, vmin, vmax, o);
    mm[0] = vmin;
    mm[1] = vmax;
    *ovf = o;
}

template <int D, typename SymT, typename OutT>
__global__ void __launch_bounds__(kR3Threads, 4) k_reconstruct_r8(const __grid_constant__ R3Params p) {
    const uint32_t lane = lane_id();
    OutT vmin = (OutT)INFINITY, vmax = (OutT)-INFINITY;
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
        // the tile's outliers: up to 32 in registers (one per lane), with the
        // chunks that need the int64 path
        const bool reg_out = r1 - r0 <= 32;
        const uint32_t nrec = reg_out ? (uint32_t)(r1 - r0) : 0u;
        uint32_t rkey = 0xFFFFFFFFu, wide_mask = 0;
        int64_t rd = 0;
        bool wide = false;
        if (reg_out) {
            if (lane < nrec) {
                rkey = (uint32_t)p.brec[2 * (r0 + lane)];
                rd = (int64_t)p.brec[2 * (r0 + lane) + 1];
                wide = rd >= (1ll << 20) || rd <= -(1ll << 20);
            }
        } else {
            for (uint64_t i = r0 + lane; i < r1; i += 32) {
                const int64_t d = (int64_t)p.brec[2 * i + 1];
                if (d >= (1ll << 20) || d <= -(1ll << 20)) wide_mask |= 1u << ((uint32_t)p.brec[2 * i] >> 8);
            }
            wide_mask = __reduce_or_sync(f3::kFull, wide_mask);
        }
        for (uint32_t m = __ballot_sync(f3::kFull, wide); m; m &= m - 1)
            wide_mask |= 1u << (__shfl_sync(f3::kFull, rkey, __ffs(m) - 1) >> 8);
        R2Chunk ch = r2_chunk_of<D>(p.g, c0);
        uint32_t cc[8];
        r2_load<D, SymT>(p, ch, lane, r2_vmask<D>(ch, lane), cc);
        for (uint64_t c = c0; c < c1; c++) {
            const uint32_t k = (uint32_t)(c - c0);
            R2Chunk nx = ch;
            uint32_t cn[8] = {};
            if (c + 1 < c1) {  // the next chunk's codes are loaded ahead
                nx = r2_chunk_of<D>(p.g, c + 1);
                r2_load<D, SymT>(p, nx, lane, r2_vmask<D>(nx, lane), cn);
            }
            if ((wide_mask >> k) & 1u) {
                OutT mmv[2] = {vmin, vmax};
                r2_chunk_wide<D, SymT, OutT>(&p, c, k, r0, r1, lane, mmv, &overflow);
                vmin = mmv[0];
                vmax = mmv[1];
            } else {
                r2_chunk<D, SymT, OutT, int32_t>(p, ch, cc, k, r0, r1, reg_out, rkey, rd, nrec, lane, vmin, vmax,
                                              overflow);
            }
            ch = nx;
#pragma unroll
            for (int j = 0; j < 8; j++) cc[j] = cn[j];
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const OutT a = __shfl_xor_sync(f3::kFull, vmin, o), b = __shfl_xor_sync(f3::kFull, vmax, o);
        vmin = fmin(vmin, a);
        vmax = fmax(vmax, b);
    }
    if (lane == 0 && vmin <= vmax) {
        atomicMin(&p.mm[0], r3_dkey((double)vmin));
        atomicMax(&p.mm[1], r3_dkey((double)vmax));
    }
    if (__any_sync(f3::kFull, overflow) && lane == 0) set_status(p.st, LZB_E_OVERFLOW);
}

}  // namespace lzb
