// K1 fast path for ChunkSpec(8,8,8): one warp per chunk, eight consecutive
// chunk ordinals per warp task ("warp tile"), persistent CTAs.  Included by
// lzb_quant.cu.  Semantics identical to the generic K1 (and to the reference,
// P/quantize.py:90-213 + P/pipeline.py:102-105 + P/codebook.py:23-27); see
// lzb_fast3d.cuh for the register layout.
//
// Per chunk: 16 elements per lane are loaded (vector loads for full chunks),
// prequantized with the guarded f64 fast path (exact fallback, int64 maths if
// any value needs it), differenced with in-register / shuffle neighbours,
// turned into codes, counted into a per-lane packed 16-bin window around the
// radius (out-of-window codes go to a shared-memory histogram), staged in
// shared memory in stream order and written back as one contiguous range.
// Outliers are ranked in stream order and stashed per warp; after its eight
// chunks the warp takes its global offset from a decoupled look-back over
// warp tiles, which keeps the records in chunk-major order.
#pragma once

#include "lzb_fast3d.cuh"

namespace lzb {

constexpr int kQ3Warps = 8;
constexpr int kQ3Threads = kQ3Warps * 32;
constexpr int kQ3TileChunks = 8;
constexpr int kQ3Stash = 32;  // outlier record slots per warp tile (overflow: re-emit pass)
constexpr int kQ3Slot = kQ3Stash;

struct Q3Params {
    const void *x;
    Geom g;
    double two_eb, inv, slack;
    float inv_hi, inv_lo;  // double-single split of inv (f32 fast path)
    int32_t r;
    uint32_t cap;
    void *codes;
    unsigned long long *hist;
    uint64_t *records;
    uint64_t out_capacity;
    lzb_dstatus *st;
    uint64_t *lb;
    unsigned int *ticket;
    uint64_t nchunks, ntiles;
    int vec_ok;  // rows of full chunks are 16-byte aligned for vector loads
    // two-phase outlier ordering: per-tile record slots + counts
    uint64_t *slots;        // ntiles * kQ3Slot records
    uint32_t *tile_cnt;     // outliers per tile
    uint32_t *over_list;    // tiles whose count exceeds kQ3Slot
    unsigned int *n_over;
    const uint64_t *tile_off;  // exclusive offsets (emit kernel)
};

template <typename InT>
struct Q3Warp {
    // per-lane state across the warp's chunks
    uint64_t hw0, hw1;  // packed 8-bit counters for codes r-8 .. r+7
    int flags;
};

template <typename SymT>
__device__ __forceinline__ void q3_hist_flush(uint64_t &hw0, uint64_t &hw1, int32_t r,
                                              uint32_t *s_hist, uint32_t lane) {
#pragma unroll
    for (int k = 0; k < 16; k++) {
        uint32_t c = (uint32_t)(((k < 8 ? hw0 : hw1) >> (8 * (k & 7))) & 0xFFu);
        uint32_t s = __reduce_add_sync(f3::kFull, c);
        if (lane == 0 && s) atomicAdd(&s_hist[r - 8 + k], s);
    }
    hw0 = hw1 = 0;
}

// Load the lane's two rows of a chunk as doubles.
template <typename InT>
__device__ __forceinline__ void q3_load(const Q3Params &p, const f3::Chunk &k, uint32_t lane,
                                        InT (&x0)[8], InT (&x1)[8]) {
    const uint32_t ly = lane & 7, lz = (lane >> 3) * 2;
    const InT *in = static_cast<const InT *>(p.x);
#pragma unroll
    for (int h = 0; h < 2; h++) {
        InT(&xr)[8] = h ? x1 : x0;
        const bool vrow = (ly < k.ey) && (lz + h < k.ez);
        const uint64_t gi = k.x0 + p.g.nx * ((k.y0 + ly) + p.g.ny * (k.z0 + lz + h));
        if (k.full && p.vec_ok) {
            if constexpr (sizeof(InT) == 4) {
                const float4 *q = reinterpret_cast<const float4 *>(in + gi);
                float4 a = __ldg(q), b = __ldg(q + 1);
                xr[0] = a.x; xr[1] = a.y; xr[2] = a.z; xr[3] = a.w;
                xr[4] = b.x; xr[5] = b.y; xr[6] = b.z; xr[7] = b.w;
            } else {
                const double2 *q = reinterpret_cast<const double2 *>(in + gi);
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    double2 a = __ldg(q + j);
                    xr[2 * j] = a.x;
                    xr[2 * j + 1] = a.y;
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < 8; j++) xr[j] = (vrow && (uint32_t)j < k.ex) ? in[gi + j] : InT(0);
        }
    }
}

constexpr uint32_t kQ3Redo = 0xFFFFFFFFu;

// Process one chunk.  emit == true: only (re)write outlier records starting at
// records[*emit_pos] (stash overflow recovery).  Returns the chunk's outlier
// count, or kQ3Redo when WIDE == false and some value needs the exact int64
// path (nothing has been written yet in that case).
template <typename InT, typename SymT, bool WIDE>
__device__ __forceinline__ uint32_t q3_chunk_body(const Q3Params &p, uint64_t c, uint32_t lane,
                                             SymT *s_codes, uint64_t *stash, uint32_t wcount,
                                             Q3Warp<InT> &w, uint32_t *s_hist, bool emit,
                                             uint64_t emit_pos, uint32_t &first_code,
                                             uint32_t &last_code) {
    const f3::Chunk k = f3::chunk_of(p.g, c);
    const uint32_t ly = lane & 7, lz0 = (lane >> 3) * 2;
    InT x0[8], x1[8];
    q3_load<InT>(p, k, lane, x0, x1);
    // validity masks of the two rows
    const uint32_t xmask = (1u << k.ex) - 1u;
    const uint32_t m0 = (ly < k.ey && lz0 < k.ez) ? xmask : 0u;
    const uint32_t m1 = (ly < k.ey && lz0 + 1 < k.ez) ? xmask : 0u;

    int32_t d0[8], d1[8];
    int64_t e0[8], e1[8];
    constexpr bool wide = WIDE;
    if (!WIDE) {
        bool ok = true;
#pragma unroll
        for (int j = 0; j < 8; j++) {
            d0[j] = f3::pq_fast((double)x0[j], p.inv, ok);
            d1[j] = f3::pq_fast((double)x1[j], p.inv, ok);
        }
        if (!__all_sync(f3::kFull, ok)) return kQ3Redo;
    }
    if (WIDE) {  // exact int64 path for the whole chunk
#pragma unroll
        for (int j = 0; j < 8; j++) {
            int fl = 0;
            e0[j] = ((m0 >> j) & 1u) ? f3::pq_exact((double)x0[j], p.two_eb, p.slack, fl) : 0;
            int fl1 = 0;
            e1[j] = ((m1 >> j) & 1u) ? f3::pq_exact((double)x1[j], p.two_eb, p.slack, fl1) : 0;
            if (!emit) w.flags |= fl | fl1;
        }
        f3::deltas<int64_t>(e0, e1, lane);
    } else {
#pragma unroll
        for (int j = 0; j < 8; j++) {
            if (!((m0 >> j) & 1u)) d0[j] = 0;
            if (!((m1 >> j) & 1u)) d1[j] = 0;
        }
        f3::deltas<int32_t>(d0, d1, lane);
    }

    // codes + outlier masks (+ window histogram)
    const int32_t r = p.r;
    uint32_t o0 = 0, o1 = 0;
    const bool win = p.cap >= 16;
#pragma unroll
    for (int h = 0; h < 2; h++) {
#pragma unroll
        for (int j = 0; j < 8; j++) {
            bool in_range;
            int64_t dd;
            if (wide) dd = h ? e1[j] : e0[j];
            else dd = h ? d1[j] : d0[j];
            int64_t ad = dd < 0 ? -dd : dd;
            in_range = ad < r;
            uint32_t code = in_range ? (uint32_t)(dd + r) : (uint32_t)r;
            const bool valid = ((h ? m1 : m0) >> j) & 1u;
            if (!emit && valid) {  // stage in stream order
                const uint32_t lz = lz0 + h;
                s_codes[k.full ? (uint32_t)j + 8 * (ly + 8 * lz) : f3::lpos(k, j, ly, lz)] = (SymT)code;
            }
            if (valid && !in_range) {
                if (h) o1 |= 1u << j; else o0 |= 1u << j;
            }
            if (!emit && valid) {
                uint32_t bin = code - (uint32_t)(r - 8);
                if (win && bin < 16u) {
                    uint64_t inc = 1ull << (8 * (bin & 7));
                    if (bin < 8) w.hw0 += inc; else w.hw1 += inc;
                } else {
                    atomicAdd(&s_hist[code], 1u);
                }
            }
        }
    }

    // outlier ranks in stream order
    uint32_t any = __ballot_sync(f3::kFull, (o0 | o1) != 0);
    uint32_t total = 0;
    if (any) {
        uint32_t r0, r1;
        const bool origin_only =
            any == 1u && __shfl_sync(f3::kFull, (o0 == 1u && o1 == 0u) ? 1 : 0, 0);
        if (origin_only) {  // the common case: the chunk origin is the only outlier
            r0 = 0;
            r1 = 1;
            total = 1;
        } else {
            f3::row_ranks(__popc(o0), __popc(o1), lane, r0, r1, total);
        }
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const uint32_t om = h ? o1 : o0;
            uint32_t rk = h ? r1 : r0;
#pragma unroll
            for (int j = 0; j < 8; j++) {  // static indices keep d/e in registers
                if (!((om >> j) & 1u)) continue;
                uint64_t gi = (k.x0 + j) + p.g.nx * ((k.y0 + ly) + p.g.ny * (k.z0 + lz0 + h));
                int64_t dd;
                if (wide) dd = h ? e1[j] : e0[j];
                else dd = h ? d1[j] : d0[j];
                if (emit) {
                    uint64_t wpos = emit_pos + rk;
                    if (wpos < p.out_capacity) {
                        p.records[2 * wpos] = gi;
                        p.records[2 * wpos + 1] = (uint64_t)dd;
                    }
                } else if (wcount + rk < (uint32_t)kQ3Stash) {
                    stash[2 * (wcount + rk)] = gi;
                    stash[2 * (wcount + rk) + 1] = (uint64_t)dd;
                }
                rk++;
            }
        }
    }
    if (emit) return total;

    // codes were staged in stream order: one contiguous write
    __syncwarp();
    const uint32_t cnt = k.ex * k.ey * k.ez;
    SymT *out = static_cast<SymT *>(p.codes) + k.base;
    if (cnt == 512 && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
        constexpr int V = 16 / sizeof(SymT);  // symbols per uint4
        const uint4 *src = reinterpret_cast<const uint4 *>(s_codes);
        uint4 *dst = reinterpret_cast<uint4 *>(out);
#pragma unroll
        for (int i = lane; i < 512 / V; i += 32) dst[i] = src[i];
    } else {
        for (uint32_t i = lane; i < cnt; i += 32) out[i] = s_codes[i];
    }
    first_code = (uint32_t)s_codes[0];
    last_code = (uint32_t)s_codes[cnt - 1];
    __syncwarp();
    return total;
}

struct Q3Res {
    uint32_t n, first, last;
    int flags;
};

// The exact int64 path lives out of line so the hot path never saves
// registers around the f64 division subroutine calls.
template <typename InT, typename SymT>
__device__ __noinline__ Q3Res q3_chunk_wide(const Q3Params *pp, uint64_t c, uint32_t lane,
                                            SymT *s_codes, uint64_t *stash, uint32_t wcount,
                                            uint32_t *s_hist, bool emit, uint64_t emit_pos) {
    const Q3Params &p = *pp;
    Q3Warp<InT> t;
    t.hw0 = t.hw1 = 0;
    t.flags = 0;
    Q3Res res;
    res.n = q3_chunk_body<InT, SymT, true>(p, c, lane, s_codes, stash, wcount, t, s_hist, emit,
                                           emit_pos, res.first, res.last);
    if (p.cap >= 16) q3_hist_flush<SymT>(t.hw0, t.hw1, p.r, s_hist, lane);
    res.flags = t.flags;
    return res;
}

template <typename InT, typename SymT>
__device__ __forceinline__ uint32_t q3_chunk(const Q3Params &p, uint64_t c, uint32_t lane,
                                             SymT *s_codes, uint64_t *stash, uint32_t wcount,
                                             Q3Warp<InT> &w, uint32_t *s_hist, bool emit,
                                             uint64_t emit_pos, uint32_t &first_code,
                                             uint32_t &last_code) {
    uint32_t n = q3_chunk_body<InT, SymT, false>(p, c, lane, s_codes, stash, wcount, w, s_hist,
                                                 emit, emit_pos, first_code, last_code);
    if (n == kQ3Redo) {
        Q3Res r = q3_chunk_wide<InT, SymT>(&p, c, lane, s_codes, stash, wcount, s_hist, emit,
                                           emit_pos);
        n = r.n;
        first_code = r.first;
        last_code = r.last;
        w.flags |= r.flags;
    }
    return n;
}

// Partial / unaligned chunks, out of line so the hot loop stays small in the
// instruction cache; the 8-bit window counters are folded before returning.
template <typename InT, typename SymT>
__device__ __noinline__ Q3Res q3_chunk_slow(const Q3Params *pp, uint64_t c, uint32_t lane,
                                            SymT *s_codes, uint64_t *stash, uint32_t wcount,
                                            uint32_t *s_hist) {
    Q3Warp<InT> t;
    t.hw0 = t.hw1 = 0;
    t.flags = 0;
    Q3Res res;
    res.n = q3_chunk<InT, SymT>(*pp, c, lane, s_codes, stash, wcount, t, s_hist, false, 0, res.first,
                                res.last);
    if (pp->cap >= 16) q3_hist_flush<SymT>(t.hw0, t.hw1, pp->r, s_hist, lane);
    res.flags = t.flags;
    return res;
}

__device__ __forceinline__ void q3_put_record(const Q3Params &p, uint64_t *stash, uint32_t wcount,
                                              bool emit, uint64_t emit_pos, uint32_t rk, uint64_t gi,
                                              int64_t dd) {
    if (emit) {
        const uint64_t wpos = emit_pos + rk;
        if (wpos < p.out_capacity) {
            p.records[2 * wpos] = gi;
            p.records[2 * wpos + 1] = (uint64_t)dd;
        }
    } else if (wcount + rk < (uint32_t)kQ3Stash) {
        stash[2 * (wcount + rk)] = gi;
        stash[2 * (wcount + rk) + 1] = (uint64_t)dd;
    }
}

// Any outlier pattern: ranks by a warp scan over rows, then each lane walks
// its outlier bits (row0 then row1, x ascending = stream order).
__device__ __forceinline__ uint32_t q3_outliers_general(const Q3Params &p, uint64_t *stash,
                                                        uint32_t wcount, bool emit, uint64_t emit_pos,
                                                        uint32_t lane, uint64_t gi0, uint64_t plane,
                                                        uint32_t o0, uint32_t o1, const int32_t (&d0)[8],
                                                        const int32_t (&d1)[8]) {
    uint32_t r0, r1, total;
    f3::row_ranks(__popc(o0), __popc(o1), lane, r0, r1, total);
    for (int h = 0; h < 2; h++) {
        uint32_t m = h ? o1 : o0, rk = h ? r1 : r0;
        while (m) {
            const uint32_t j = __ffs(m) - 1;
            m &= m - 1;
            int32_t dd = h ? d1[0] : d0[0];  // select without dynamic indexing
#pragma unroll
            for (int k = 1; k < 8; k++) dd = (j == (uint32_t)k) ? (h ? d1[k] : d0[k]) : dd;
            q3_put_record(p, stash, wcount, emit, emit_pos, rk++, gi0 + (h ? plane : 0) + j, dd);
        }
    }
    return total;
}

// Lean path for a FULL 8x8x8 chunk: no masks, no divisions.  The lane's two
// input rows were prefetched into shared memory (`stg`, cp.async) one chunk
// ahead.  gi0 = global index of this lane's row0 start, sbase = stream offset
// of the chunk.  Returns kQ3Redo (nothing written) when a value needs the
// exact path.  Histogram: the 16 codes around the radius go to this lane's
// private column of a per-warp shared table (conflict-free red.shared), the
// rest to the CTA table.
template <typename InT, typename SymT>
__device__ __forceinline__ uint32_t q3_full(const Q3Params &p, const InT *stg, uint64_t gi0,
                                            uint64_t sbase, uint32_t lane, uint64_t *stash,
                                            uint32_t wcount, uint32_t colbase, uint32_t hbase,
                                            bool emit, uint64_t emit_pos) {
    const uint32_t ly = lane & 7, lz0 = (lane >> 3) * 2;
    const uint64_t plane = p.g.nx * p.g.ny;
    int32_t d0[8], d1[8];
    bool ok = true;
    if constexpr (sizeof(InT) == 4) {
        const float4 *q = reinterpret_cast<const float4 *>(stg);
        float4 a = q[0], b = q[32], c = q[64], d = q[96];
        float x0[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        float x1[8] = {c.x, c.y, c.z, c.w, d.x, d.y, d.z, d.w};
#pragma unroll
        for (int j = 0; j < 8; j++) {
            d0[j] = f3::pq_fast_f32(x0[j], p.inv_hi, p.inv_lo, ok);
            d1[j] = f3::pq_fast_f32(x1[j], p.inv_hi, p.inv_lo, ok);
        }
    } else {
        const double2 *q = reinterpret_cast<const double2 *>(stg);
#pragma unroll
        for (int j = 0; j < 4; j++) {
            double2 a = q[32 * j], b = q[32 * (4 + j)];
            d0[2 * j] = f3::pq_fast(a.x, p.inv, ok);
            d0[2 * j + 1] = f3::pq_fast(a.y, p.inv, ok);
            d1[2 * j] = f3::pq_fast(b.x, p.inv, ok);
            d1[2 * j + 1] = f3::pq_fast(b.y, p.inv, ok);
        }
    }
    if (!__all_sync(f3::kFull, ok)) return kQ3Redo;
    f3::deltas<int32_t>(d0, d1, lane);

    const int32_t r = p.r;
    // window of private columns: codes r-8 .. r+7 (none when cap < 16)
    const uint32_t klo = p.cap >= 16 ? (uint32_t)(r - 8) : (uint32_t)(r + 16);
    uint32_t o0 = 0, o1 = 0;
    uint32_t c0[8], c1[8];
#pragma unroll
    for (int j = 0; j < 8; j++) {
        const bool i0 = (uint32_t)(d0[j] + r - 1) < (uint32_t)(2 * r - 1);  // |d| < r
        const bool i1 = (uint32_t)(d1[j] + r - 1) < (uint32_t)(2 * r - 1);
        c0[j] = i0 ? (uint32_t)(d0[j] + r) : (uint32_t)r;
        c1[j] = i1 ? (uint32_t)(d1[j] + r) : (uint32_t)r;
        o0 |= (uint32_t)!i0 << j;
        o1 |= (uint32_t)!i1 << j;
    }
    // outliers: ranks in stream order.  Common case: only the chunk origin
    // (lane 0, row 0, x 0) -- one record written by lane 0.
    const uint32_t any = __ballot_sync(f3::kFull, (o0 | o1) != 0);
    uint32_t total = 0;
    if (any) {
        const bool origin_only =
            any == 1u && __shfl_sync(f3::kFull, (o0 == 1u && o1 == 0u) ? 1 : 0, 0);
        if (origin_only) {
            total = 1;
            if (lane == 0) q3_put_record(p, stash, wcount, emit, emit_pos, 0, gi0, d0[0]);
        } else {
            total = q3_outliers_general(p, stash, wcount, emit, emit_pos, lane, gi0, plane, o0, o1,
                                        d0, d1);
        }
    }
    if (emit) return total;

    // histogram (fire-and-forget shared-memory reductions)
#pragma unroll
    for (int h = 0; h < 2; h++) {
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const uint32_t code = h ? c1[j] : c0[j];
            const uint32_t key = code - klo;
            const uint32_t addr = key < 16u ? colbase + (key << 7) : hbase + (code << 2);
            asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(addr) : "memory");
        }
    }

    // codes: each row is 8 consecutive stream symbols -> one vector store
    SymT *out = static_cast<SymT *>(p.codes) + sbase;
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const uint32_t(&cr)[8] = h ? c1 : c0;
        SymT *dst = out + 8 * (ly + 8 * (lz0 + h));
        if constexpr (sizeof(SymT) == 2) {
            uint4 v;
            v.x = cr[0] | (cr[1] << 16);
            v.y = cr[2] | (cr[3] << 16);
            v.z = cr[4] | (cr[5] << 16);
            v.w = cr[6] | (cr[7] << 16);
            *reinterpret_cast<uint4 *>(dst) = v;
        } else {
            reinterpret_cast<uint4 *>(dst)[0] = make_uint4(cr[0], cr[1], cr[2], cr[3]);
            reinterpret_cast<uint4 *>(dst)[1] = make_uint4(cr[4], cr[5], cr[6], cr[7]);
        }
    }
    return total;
}

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void *g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// chunk c of the fast grid: full? + lane row0 global index + stream offset
// Location of chunk (bx, by, bz) of the fast grid: full?, the lane's row0
// global index and the chunk's stream offset (meaningful for full chunks,
// where the stream offset is nx*ny*8*bz + nx*64*by + 512*bx).  Along a chunk
// row the next location is an increment (q3_next).
struct Q3Loc {
    bool full, row_full;
    uint64_t gi0, sbase;
};

__device__ __forceinline__ Q3Loc q3_loc(const Q3Params &p, uint64_t bx, uint64_t by, uint64_t bz,
                                        uint64_t lane_off) {
    Q3Loc l;
    l.row_full = p.vec_ok && (by * 8 + 8 <= p.g.ny) && (bz * 8 + 8 <= p.g.nz);
    l.full = l.row_full && (bx * 8 + 8 <= p.g.nx);
    l.sbase = p.g.nx * p.g.ny * 8 * bz + p.g.nx * 64 * by + 512 * bx;
    l.gi0 = bx * 8 + p.g.nx * (by * 8 + p.g.ny * (bz * 8)) + lane_off;
    return l;
}

// the lane copies its two rows (2 x 8 values) into its stage slot
template <typename InT>
__device__ __forceinline__ void q3_prefetch(const Q3Params &p, const Q3Loc &l, uint32_t saddr) {
    const InT *in = static_cast<const InT *>(p.x);
    const InT *r0 = in + l.gi0;
    const InT *r1 = r0 + p.g.nx * p.g.ny;
    constexpr int V = 16 / sizeof(InT);  // values per 16-byte copy
#pragma unroll
    for (int k = 0; k < 8 / V; k++) {  // piece-major: conflict-free 16-byte reads
        cp_async16(saddr + 512 * k, r0 + V * k);
        cp_async16(saddr + 512 * (8 / V + k), r1 + V * k);
    }
}

template <typename InT, typename SymT>
__global__ void __launch_bounds__(kQ3Threads, 2) k_quantize3d8(const __grid_constant__ Q3Params p) {
    extern __shared__ __align__(16) unsigned char q3_smem[];
    // [stage: warps x 2 x 32 lanes x 16 values][s_codes: warps x 512 SymT]
    // [s_col: warps x 16 bins x 32 lanes u32][s_hist: cap u32]
    constexpr uint32_t kLaneStage = 16 * sizeof(InT);
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    unsigned char *stage = q3_smem + warp * 2 * 32 * kLaneStage;
    unsigned char *after_stage = q3_smem + kQ3Warps * 2 * 32 * kLaneStage;
    SymT *s_codes = reinterpret_cast<SymT *>(after_stage) + warp * 512;
    uint32_t *s_col = reinterpret_cast<uint32_t *>(after_stage + kQ3Warps * 512 * sizeof(SymT));
    uint32_t *s_hist = s_col + kQ3Warps * 16 * 32;
    for (uint32_t i = threadIdx.x; i < kQ3Warps * 16 * 32; i += blockDim.x) s_col[i] = 0;
    for (uint32_t i = threadIdx.x; i < p.cap; i += blockDim.x) s_hist[i] = 0;
    __syncthreads();
    const uint32_t stage_s = (uint32_t)__cvta_generic_to_shared(stage) + lane * 16;
    const uint64_t lane_off = p.g.nx * ((lane & 7) + p.g.ny * ((lane >> 3) * 2));
    const uint32_t hbase = (uint32_t)__cvta_generic_to_shared(s_hist);
    // codes outside the 16-bin window (or books with cap < 16) go straight to s_hist
    const uint32_t colbase = p.cap >= 16
        ? (uint32_t)__cvta_generic_to_shared(s_col + warp * 16 * 32) + lane * 4
        : 0xFFFFFFFFu;

    Q3Warp<InT> w;
    w.hw0 = w.hw1 = 0;
    w.flags = 0;
    // Tiles are claimed one ahead so the first chunk of the next tile is
    // prefetched while the last chunk of the current one is processed.
    // Tickets hand out tiles from the END of the stream: the last chunk
    // layer / row ends are the partial chunks (exact path, several times
    // slower), so they start first and the run ends on full tiles instead of
    // a tail of a few warps on partial ones.  Tiles are independent.
    auto claim = [&]() -> uint64_t {
        uint64_t t = 0;
        if (lane == 0) t = atomicAdd(p.ticket, 1u);
        t = __shfl_sync(f3::kFull, t, 0);
        return t < p.ntiles ? p.ntiles - 1 - t : p.ntiles;
    };
    uint64_t t = claim();
    uint64_t t_next = t < p.ntiles ? claim() : p.ntiles;
    uint32_t bx = 0, by = 0, bz = 0;
    auto tile_origin = [&](uint64_t tt) {
        const uint64_t c0 = tt * kQ3TileChunks;
        const uint64_t rowc = c0 / p.g.nbx;
        bx = (uint32_t)(c0 - rowc * p.g.nbx);
        by = (uint32_t)(rowc % p.g.nby);
        bz = (uint32_t)(rowc / p.g.nby);
    };
    Q3Loc cur;
    cur.full = false;
    if (t < p.ntiles) {
        tile_origin(t);
        cur = q3_loc(p, bx, by, bz, lane_off);
        if (cur.full) q3_prefetch<InT>(p, cur, stage_s);
    }
    cp_async_commit();
    uint32_t sb = 0;
    while (t < p.ntiles) {
        const uint64_t c0 = t * kQ3TileChunks;
        const uint32_t nk = (uint32_t)(umin64(c0 + kQ3TileChunks, p.nchunks) - c0);
        uint64_t *slot = p.slots + t * 2 * kQ3Slot;
        uint32_t wcount = 0;
        for (uint32_t k = 0; k < nk; k++) {
            // the next chunk: same tile, else the first chunk of the next tile
            Q3Loc nxt = cur;
            bool have_next = true;
            if (k + 1 < nk) {
                if (++bx < (uint32_t)p.g.nbx) {  // same chunk row: increment
                    nxt.gi0 += 8;
                    nxt.sbase += 512;
                    nxt.full = nxt.row_full && (bx * 8 + 8 <= p.g.nx);
                } else {
                    bx = 0;
                    if (++by == (uint32_t)p.g.nby) {
                        by = 0;
                        ++bz;
                    }
                    nxt = q3_loc(p, bx, by, bz, lane_off);
                }
            } else if (t_next < p.ntiles) {
                tile_origin(t_next);
                nxt = q3_loc(p, bx, by, bz, lane_off);
            } else {
                have_next = false;
                nxt.full = false;
            }
            if (have_next && nxt.full) q3_prefetch<InT>(p, nxt, stage_s + (sb ^ 1) * 32 * kLaneStage);
            cp_async_commit();
            cp_async_wait1();  // this chunk's rows have landed
            uint32_t n = kQ3Redo;
            if (cur.full)
                n = q3_full<InT, SymT>(p, reinterpret_cast<const InT *>(stage + sb * 32 * kLaneStage + lane * 16),
                                       cur.gi0, cur.sbase, lane, slot, wcount, colbase, hbase, false, 0);
            if (n == kQ3Redo) {
                const Q3Res rr = q3_chunk_slow<InT, SymT>(&p, c0 + k, lane, s_codes, slot, wcount, s_hist);
                n = rr.n;
                w.flags |= rr.flags;
            }
            wcount += n;
            cur = nxt;
            sb ^= 1;
        }
        if (lane == 0) {
            p.tile_cnt[t] = wcount;
            if (wcount > (uint32_t)kQ3Slot) p.over_list[atomicAdd(p.n_over, 1u)] = (uint32_t)t;
        }
        t = t_next;
        if (t < p.ntiles) t_next = claim();
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    // fold this warp's private columns into the CTA histogram
    if (p.cap >= 16) {
#pragma unroll
        for (int k = 0; k < 16; k++) {
            const uint32_t v = __reduce_add_sync(f3::kFull, s_col[(warp * 16 + k) * 32 + lane]);
            if (lane == 0 && v) atomicAdd(&s_hist[p.r - 8 + k], v);
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < p.cap; i += blockDim.x)
        if (s_hist[i]) atomicAdd(&p.hist[i], (unsigned long long)s_hist[i]);
    int flags = __reduce_or_sync(f3::kFull, w.flags);
    if (lane == 0 && flags) set_status(p.st, (flags & 1) ? LZB_E_OVERFLOW : LZB_E_ASSERT);
}

// Phase 2a: copy each tile's slot records to its final (chunk-major) place.
__global__ void k_q3_compact(const __grid_constant__ Q3Params p) {
    const uint32_t lane = lane_id();
    const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t t = gw; t < p.ntiles; t += nw) {
        const uint32_t n = p.tile_cnt[t];
        if (n == 0 || n > (uint32_t)kQ3Slot) continue;
        const uint64_t o = p.tile_off[t];
        for (uint32_t i = lane; i < n; i += 32) {
            if (o + i < p.out_capacity) {
                p.records[2 * (o + i)] = p.slots[(t * kQ3Slot + i) * 2];
                p.records[2 * (o + i) + 1] = p.slots[(t * kQ3Slot + i) * 2 + 1];
            }
        }
    }
}

// Phase 2b: tiles that overflowed their slots re-derive their outliers and
// write them straight to the final positions (noisy data only).
template <typename InT, typename SymT>
__global__ void __launch_bounds__(kQ3Threads) k_q3_emit(const __grid_constant__ Q3Params p) {
    extern __shared__ __align__(16) unsigned char q3e_smem[];
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    SymT *s_codes = reinterpret_cast<SymT *>(q3e_smem) + warp * 512;
    const uint32_t nover = *p.n_over;
    Q3Warp<InT> w;
    w.hw0 = w.hw1 = 0;
    w.flags = 0;
    const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t i = gw; i < nover; i += nw) {
        const uint64_t t = p.over_list[i];
        const uint64_t c0 = t * kQ3TileChunks;
        const uint64_t c1 = umin64(c0 + kQ3TileChunks, p.nchunks);
        uint64_t pos = p.tile_off[t];
        for (uint64_t c = c0; c < c1; c++) {
            uint32_t f, l;
            pos += q3_chunk<InT, SymT>(p, c, lane, s_codes, nullptr, 0, w, nullptr, true, pos, f, l);
        }
    }
}

// exclusive scan of the tile counts (single pass, look-back) + totals
__global__ void __launch_bounds__(256) k_q3_scan(const __grid_constant__ Q3Params p,
                                                 uint64_t *tile_off, uint64_t *lb,
                                                 unsigned int *ticket) {
    __shared__ uint64_t s_t, s_ex;
    __shared__ uint64_t s_scan[33];
    const uint64_t n = p.ntiles;
    const uint64_t ntl = (n + 2047) / 2048;
    while (true) {
        if (threadIdx.x == 0) s_t = atomicAdd(ticket, 1u);
        __syncthreads();
        const uint64_t t = s_t;
        if (t >= ntl) break;
        const uint64_t base = t * 2048 + threadIdx.x * 8;
        uint64_t v[8], sum = 0;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            v[k] = base + k < n ? p.tile_cnt[base + k] : 0;
            sum += v[k];
        }
        uint64_t tot;
        uint64_t off = block_exclusive_scan<uint64_t>(sum, s_scan, &tot);
        if ((threadIdx.x >> 5) == 0) {
            uint64_t ex = lookback_warp(lb, t, tot);
            if (lane_id() == 0) s_ex = ex;
        }
        __syncthreads();
        uint64_t run = s_ex + off;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            if (base + k < n) tile_off[base + k] = run;
            run += v[k];
        }
        if (t == ntl - 1 && threadIdx.x == 0) {
            p.st->u[0] = s_ex + tot;
            if (s_ex + tot > p.out_capacity) set_status(p.st, LZB_E_CAPACITY);
        }
        __syncthreads();
    }
}

}  // namespace lzb
