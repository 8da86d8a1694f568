// K1 for 2D fields with ChunkSpec(16,16) and 1D fields with ChunkSpec(256):
// one warp per 256-element chunk, eight per lane, eight consecutive chunk
// ordinals per warp task ("warp tile"), persistent CTAs.
// Included by lzb_quant.cu.  Semantics identical to the generic K1 and to the
// reference (P/quantize.py:90-213, P/pipeline.py:102-105,
// P/codebook.py:23-27); the outlier hand-off (per-tile slots, k_q3_scan,
// k_q3_compact, overflow re-emission) is the 3D fast path's.
//
// Register layout (D = 2): lane l owns row ly = l >> 1 of the chunk and the
// eight x-elements xh = 8 * (l & 1) .. xh + 7; (D = 1) lane l owns elements
// 8 l .. 8 l + 7.  The chunk's stream position of element j is then
// ly * ex + xh + j, resp. 8 l + j (8 l + j for every full chunk), so a lane's
// eight codes are one 16-byte store and the warp's 256 codes one contiguous
// 512-byte range.  1D: d = q - (left neighbour), in-lane or lane l - 1's last
// element.  2D: the Lorenzo delta is separable,
//   d = dx(dy(q)):  dy needs the row above = lane l - 2 (shfl by 2),
//                   dx the element to the left = in-lane, or the last
//                   element of lane l - 1 for the right half (shfl by 1),
// with everything outside the (clipped) chunk zero (P/quantize.py:136-141).
#pragma once

#include "lzb_quant3d.cuh"

namespace lzb {

struct Q2Chunk {
    uint64_t x0, y0, base;
    uint32_t ex, ey;
    bool full;
};

template <int D>
__device__ __forceinline__ Q2Chunk q2_chunk_of(const Geom &g, uint64_t c) {
    Q2Chunk k;
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
        k.base = g.nx * 16 * by + (uint64_t)k.ey * 16 * bx;  // rows above + full chunks to the left
    }
    return k;
}

// global index / chunk stream position of the lane's first element
template <int D>
__device__ __forceinline__ uint64_t q2_lane_gi(const Q2Chunk &k, uint32_t lane, uint64_t nx) {
    if constexpr (D == 1) return k.x0 + 8 * lane;
    else return (k.x0 + 8 * (lane & 1)) + nx * (k.y0 + (lane >> 1));
}
template <int D>
__device__ __forceinline__ uint32_t q2_lane_pos(const Q2Chunk &k, uint32_t lane) {
    if constexpr (D == 1) return 8 * lane;
    else return (lane >> 1) * k.ex + 8 * (lane & 1);
}

// Lorenzo deltas of the lane's eight values (int32 or int64)
template <int D, typename I>
__device__ __forceinline__ void q2_deltas(I (&v)[8], uint32_t lane) {
    if constexpr (D == 2) {
        const bool top = lane < 2;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const I up = __shfl_up_sync(f3::kFull, v[j], 2);
            v[j] -= top ? (I)0 : up;
        }
    }
    const bool has_left = D == 1 ? lane > 0 : (lane & 1) != 0;
    const I left = __shfl_up_sync(f3::kFull, v[7], 1);
#pragma unroll
    for (int j = 7; j > 0; j--) v[j] -= v[j - 1];
    v[0] -= has_left ? left : (I)0;
}

// Outlier ranks in stream order: lanes in order, then x within the lane.
__device__ __forceinline__ uint32_t q2_rank(uint32_t om, uint32_t lane, uint32_t &total) {
    const uint32_t c = __popc(om);
    uint32_t inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t a = __shfl_up_sync(f3::kFull, inc, o);
        if (lane >= (uint32_t)o) inc += a;
    }
    total = __shfl_sync(f3::kFull, inc, 31);
    return inc - c;
}

template <int D, typename I>
__device__ __forceinline__ void q2_records(const Q3Params &p, const Q2Chunk &k, uint32_t lane, uint32_t om,
                                           uint32_t rk, const I (&d)[8], uint64_t *stash, uint32_t wcount,
                                           bool emit, uint64_t emit_pos) {
    const uint64_t gi0 = q2_lane_gi<D>(k, lane, p.g.nx);
#pragma unroll
    for (int j = 0; j < 8; j++) {
        if (!((om >> j) & 1u)) continue;
        q3_put_record(p, stash, wcount, emit, emit_pos, rk++, gi0 + j, (int64_t)d[j]);
    }
}

// codes of one chunk: store + histogram (not in emit mode)
template <int D, typename SymT>
__device__ __forceinline__ void q2_codes(const Q3Params &p, const Q2Chunk &k, uint32_t lane, uint32_t vmask,
                                         const uint32_t (&c)[8], uint32_t colbase, uint32_t hbase) {
    const uint32_t klo = p.cap >= 16 ? (uint32_t)(p.r - 8) : (uint32_t)(p.r + 16);
#pragma unroll
    for (int j = 0; j < 8; j++) {
        if (!((vmask >> j) & 1u)) continue;
        const uint32_t key = c[j] - klo;
        const uint32_t addr = key < 16u ? colbase + (key << 7) : hbase + (c[j] << 2);
        asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory");
    }
    SymT *out = static_cast<SymT *>(p.codes) + k.base;
    if (k.full) {
        SymT *dst = out + 8 * lane;
        if constexpr (sizeof(SymT) == 2) {
            uint4 v;
            v.x = c[0] | (c[1] << 16);
            v.y = c[2] | (c[3] << 16);
            v.z = c[4] | (c[5] << 16);
            v.w = c[6] | (c[7] << 16);
            *reinterpret_cast<uint4 *>(dst) = v;
        } else {
            reinterpret_cast<uint4 *>(dst)[0] = make_uint4(c[0], c[1], c[2], c[3]);
            reinterpret_cast<uint4 *>(dst)[1] = make_uint4(c[4], c[5], c[6], c[7]);
        }
    } else {
        const uint32_t pos0 = q2_lane_pos<D>(k, lane);
#pragma unroll
        for (int j = 0; j < 8; j++)
            if ((vmask >> j) & 1u) out[pos0 + j] = (SymT)c[j];
    }
}

// valid elements of the lane in chunk k
template <int D>
__device__ __forceinline__ uint32_t q2_vmask(const Q2Chunk &k, uint32_t lane) {
    const uint32_t xh = D == 1 ? 8 * lane : 8 * (lane & 1), ly = D == 1 ? 0u : lane >> 1;
    if (ly >= k.ey || xh >= k.ex) return 0u;
    const uint32_t w = k.ex - xh;
    return w >= 8 ? 0xFFu : ((1u << w) - 1u);
}

template <int D, typename InT>
__device__ __forceinline__ void q2_load(const Q3Params &p, const Q2Chunk &k, uint32_t lane, uint32_t vmask,
                                        InT (&x)[8]) {
    const InT *in = static_cast<const InT *>(p.x) + q2_lane_gi<D>(k, lane, p.g.nx);
    if (k.full && p.vec_ok) {
        if constexpr (sizeof(InT) == 4) {
            const float4 a = __ldg(reinterpret_cast<const float4 *>(in));
            const float4 b = __ldg(reinterpret_cast<const float4 *>(in) + 1);
            x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
            x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
        } else {
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const double2 a = __ldg(reinterpret_cast<const double2 *>(in) + j);
                x[2 * j] = a.x;
                x[2 * j + 1] = a.y;
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < 8; j++) x[j] = ((vmask >> j) & 1u) ? in[j] : InT(0);
    }
}

// The exact int64 path (a value needs the reference's f64 division), out of
// line: the whole chunk is redone from its input.
template <int D, typename InT, typename SymT>
__device__ __noinline__ uint32_t q2_chunk_wide(const Q3Params *pp, uint64_t c, uint32_t lane, uint64_t *stash,
                                               uint32_t wcount, uint32_t colbase, uint32_t hbase, bool emit,
                                               uint64_t emit_pos, int *flags) {
    const Q3Params &p = *pp;
    const Q2Chunk k = q2_chunk_of<D>(p.g, c);
    const uint32_t vm = q2_vmask<D>(k, lane);
    InT x[8];
    q2_load<D, InT>(p, k, lane, vm, x);
    int64_t d[8];
    int fl = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) d[j] = ((vm >> j) & 1u) ? f3::pq_exact((double)x[j], p.two_eb, p.slack, fl) : 0;
    if (!emit) *flags |= fl;
    q2_deltas<D, int64_t>(d, lane);
    uint32_t cc[8], om = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) {
        const int64_t ad = d[j] < 0 ? -d[j] : d[j];
        const bool in = ad < p.r;
        cc[j] = in ? (uint32_t)(d[j] + p.r) : (uint32_t)p.r;
        om |= (uint32_t)(!in && ((vm >> j) & 1u)) << j;
    }
    uint32_t total;
    const uint32_t rk = q2_rank(om, lane, total);
    if (om) q2_records<D, int64_t>(p, k, lane, om, rk, d, stash, wcount, emit, emit_pos);
    if (!emit) q2_codes<D, SymT>(p, k, lane, vm, cc, colbase, hbase);
    return total;
}

// One chunk from its (already loaded) values; returns the outlier count.
template <int D, typename InT, typename SymT>
__device__ __forceinline__ uint32_t q2_chunk(const Q3Params &p, uint64_t c, const Q2Chunk &k, const InT (&x)[8],
                                             uint32_t lane, uint64_t *stash, uint32_t wcount, uint32_t colbase,
                                             uint32_t hbase, bool emit, uint64_t emit_pos, int &flags) {
    const uint32_t vm = q2_vmask<D>(k, lane);
    int32_t d[8];
    bool ok = true;
#pragma unroll
    for (int j = 0; j < 8; j++) {
        int32_t v;
        if constexpr (sizeof(InT) == 4) v = f3::pq_fast_f32(x[j], p.inv_hi, p.inv_lo, ok);
        else v = f3::pq_fast(x[j], p.inv, ok);
        d[j] = ((vm >> j) & 1u) ? v : 0;
    }
    if (!__all_sync(f3::kFull, ok))
        return q2_chunk_wide<D, InT, SymT>(&p, c, lane, stash, wcount, colbase, hbase, emit, emit_pos, &flags);
    q2_deltas<D, int32_t>(d, lane);
    const int32_t r = p.r;
    uint32_t cc[8], om = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) {
        const bool in = (uint32_t)(d[j] + r - 1) < (uint32_t)(2 * r - 1);  // |d| < r
        cc[j] = in ? (uint32_t)(d[j] + r) : (uint32_t)r;
        om |= (uint32_t)!in << j;
    }
    om &= vm;
    const uint32_t any = __ballot_sync(f3::kFull, om != 0);
    uint32_t total = 0;
    if (any) {
        const uint32_t rk = q2_rank(om, lane, total);
        if (om) q2_records<D, int32_t>(p, k, lane, om, rk, d, stash, wcount, emit, emit_pos);
    }
    if (!emit) q2_codes<D, SymT>(p, k, lane, vm, cc, colbase, hbase);
    return total;
}

template <int D, typename InT, typename SymT>
__global__ void __launch_bounds__(kQ3Threads, 4) k_quantize_r8(const __grid_constant__ Q3Params p) {
    extern __shared__ __align__(16) unsigned char q2_smem[];
    // [s_col: warps x 16 bins x 32 lanes u32][s_hist: cap u32]
    uint32_t *s_col = reinterpret_cast<uint32_t *>(q2_smem);
    uint32_t *s_hist = s_col + kQ3Warps * 16 * 32;
    for (uint32_t i = threadIdx.x; i < kQ3Warps * 16 * 32; i += blockDim.x) s_col[i] = 0;
    for (uint32_t i = threadIdx.x; i < p.cap; i += blockDim.x) s_hist[i] = 0;
    __syncthreads();
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    const uint32_t hbase = (uint32_t)__cvta_generic_to_shared(s_hist);
    const uint32_t colbase = p.cap >= 16
        ? (uint32_t)__cvta_generic_to_shared(s_col + warp * 16 * 32) + lane * 4
        : 0xFFFFFFFFu;
    int flags = 0;
    // tiles from the end of the stream first (partial chunks; see k_quantize3d8)
    auto claim = [&]() -> uint64_t {
        uint64_t t = 0;
        if (lane == 0) t = atomicAdd(p.ticket, 1u);
        t = __shfl_sync(f3::kFull, t, 0);
        return t < p.ntiles ? p.ntiles - 1 - t : p.ntiles;
    };
    // the next chunk's values are loaded while the current one is processed
    uint64_t t = claim();
    Q2Chunk k{};
    InT x[8] = {};
    if (t < p.ntiles) {
        k = q2_chunk_of<D>(p.g, t * kQ3TileChunks);
        q2_load<D, InT>(p, k, lane, q2_vmask<D>(k, lane), x);
    }
    while (t < p.ntiles) {
        const uint64_t c0 = t * kQ3TileChunks;
        const uint64_t c1 = umin64(c0 + kQ3TileChunks, p.nchunks);
        uint64_t *slot = p.slots + t * 2 * kQ3Slot;
        uint32_t wcount = 0;
        uint64_t t_next = p.ntiles;
        for (uint64_t c = c0; c < c1; c++) {
            uint64_t cn = c + 1;
            if (cn == c1) {  // the first chunk of the warp's next tile
                t_next = claim();
                cn = t_next < p.ntiles ? t_next * kQ3TileChunks : p.nchunks;
            }
            Q2Chunk kn = k;
            InT xn[8] = {};
            if (cn < p.nchunks) {
                kn = q2_chunk_of<D>(p.g, cn);
                q2_load<D, InT>(p, kn, lane, q2_vmask<D>(kn, lane), xn);
            }
            wcount += q2_chunk<D, InT, SymT>(p, c, k, x, lane, slot, wcount, colbase, hbase, false, 0, flags);
            k = kn;
#pragma unroll
            for (int j = 0; j < 8; j++) x[j] = xn[j];
        }
        if (lane == 0) {
            p.tile_cnt[t] = wcount;
            if (wcount > (uint32_t)kQ3Slot) p.over_list[atomicAdd(p.n_over, 1u)] = (uint32_t)t;
        }
        t = t_next;
    }
    __syncwarp();
    if (p.cap >= 16) {
#pragma unroll
        for (int b = 0; b < 16; b++) {
            const uint32_t v = __reduce_add_sync(f3::kFull, s_col[(warp * 16 + b) * 32 + lane]);
            if (lane == 0 && v) atomicAdd(&s_hist[p.r - 8 + b], v);
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < p.cap; i += blockDim.x)
        if (s_hist[i]) atomicAdd(&p.hist[i], (unsigned long long)s_hist[i]);
    flags = __reduce_or_sync(f3::kFull, flags);
    if (lane == 0 && flags) set_status(p.st, (flags & 1) ? LZB_E_OVERFLOW : LZB_E_ASSERT);
}

// Tiles that overflowed their slots re-derive their outliers straight into
// the final positions (noisy data only).
template <int D, typename InT, typename SymT>
__global__ void __launch_bounds__(kQ3Threads) k_q2_emit(const __grid_constant__ Q3Params p) {
    const uint32_t lane = lane_id();
    const uint32_t nover = *p.n_over;
    int flags = 0;
    const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t i = gw; i < nover; i += nw) {
        const uint64_t t = p.over_list[i];
        const uint64_t c0 = t * kQ3TileChunks;
        const uint64_t c1 = umin64(c0 + kQ3TileChunks, p.nchunks);
        uint64_t pos = p.tile_off[t];
        for (uint64_t c = c0; c < c1; c++) {
            const Q2Chunk k = q2_chunk_of<D>(p.g, c);
            InT x[8];
            q2_load<D, InT>(p, k, lane, q2_vmask<D>(k, lane), x);
            pos += q2_chunk<D, InT, SymT>(p, c, k, x, lane, nullptr, 0, 0, 0, true, pos, flags);
        }
    }
}

}  // namespace lzb
