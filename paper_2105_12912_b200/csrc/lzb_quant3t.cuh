// K1 TMA path for ChunkSpec(8,8,8), f32 input, u16 codes (the C5 workload).
// Included by lzb_quant.cu after lzb_quant3d.cuh.  Semantics identical to the
// reference (P/quantize.py:90-213, P/pipeline.py:102-105, P/codebook.py:23-27)
// and to k_quantize3d8; see lzb_fast3d.cuh for the per-chunk register layout.
//
// A super tile is 16 consecutive chunks along x = a 128x8x8 f32 box (32 KB,
// 512-byte row segments; two outlier tiles of 8 chunks).  Each persistent
// CTA (16 warps, one per SM) owns super tiles b, b + G, b + 2G, ... and
// streams them through a ring of kT1Stages shared-memory stages with TMA
// (four 32x8x8 boxes per tile, SWIZZLE_128B so the warps' 16-byte row reads
// are bank-conflict free), completion tracked by one mbarrier per stage.
// Each warp takes one chunk of the tile: prequant (f32 double-single fast
// path, exact f64 division only for the rare element near a rounding tie),
// Lorenzo deltas in registers/shuffles, codes stored as 16-byte rows straight
// into the chunk-major stream, histogram into per-lane shared columns.  No
// CTA barrier per tile: warps leave their outlier counts / first records in
// the stage's slots and arrive on the stage's named barrier; one rotating
// publisher warp syncs on it, publishes the two outlier tiles and issues the
// stage's TMA refill.
// (Measured alternatives that were slower on C5q: 2 or 4 stages, 8-chunk
// tiles with 2 CTAs/SM, releasing the stage right after the shared-memory
// reads -- more TMA traffic in flight costs more than it hides.)
#pragma once

#include <cudaTypedefs.h>

namespace lzb {

constexpr int kT1Warps = 16;       // one chunk of the super tile per warp
constexpr int kT1Threads = kT1Warps * 32;
constexpr int kT1Stages = 3;       // tiles in flight per CTA (measured: 2 / 3 / 4 stages -> 3.97 / 3.75 / 3.85 ms on C5q)
constexpr uint32_t kT1Box = 8192;  // bytes per 32x8x8 f32 box
constexpr uint32_t kT1Tile = 4 * kT1Box;  // 16 chunks = 128x8x8 f32 (512-byte rows)

struct T1Params {
    Q3Params q;
    uint32_t tpr;               // super tiles (16 chunks) per chunk row (nbx / 16)
    uint32_t step_q, step_rem;  // divmod(gridDim.x, tpr)
    uint64_t nst;               // super tiles (= 2 outlier tiles of kQ3TileChunks each)
};

__device__ __forceinline__ void t1_mbar_init(uint32_t a, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void t1_mbar_expect(uint32_t a, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void t1_mbar_wait(uint32_t a, uint32_t parity) {
    uint32_t ok = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!ok);
}
__device__ __forceinline__ void t1_tma3(uint32_t dst, const CUtensorMap *map, int x, int y, int z, uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(mbar)
        : "memory");
}

constexpr int kT1Sub = 4;  // records kept per chunk (more: the tile is re-emitted by k_q3_emit)

// Tile position: tile column tx (8 chunks) in chunk row (by, bz).  The
// persistent loop steps by G tiles; (q, rem) = divmod(G, tiles per row).
struct T1Pos {
    uint32_t tx, by, bz;
};
__device__ __forceinline__ T1Pos t1_pos(const T1Params &P, uint64_t t) {
    T1Pos o;
    const uint32_t row = (uint32_t)(t / P.tpr);
    o.tx = (uint32_t)(t - (uint64_t)row * P.tpr);
    o.by = row % P.q.g.nby;
    o.bz = row / P.q.g.nby;
    return o;
}
__device__ __forceinline__ void t1_step(const T1Params &P, T1Pos &o) {
    o.tx += P.step_rem;
    o.by += P.step_q;
    if (o.tx >= P.tpr) {
        o.tx -= P.tpr;
        o.by++;
    }
    if (o.by >= (uint32_t)P.q.g.nby) {
        o.bz += o.by / (uint32_t)P.q.g.nby;
        o.by %= (uint32_t)P.q.g.nby;
    }
}
__device__ __forceinline__ void t1_issue(const CUtensorMap *map, const T1Pos &o, uint32_t dst, uint32_t mbar) {
    t1_mbar_expect(mbar, kT1Tile);
#pragma unroll
    for (int b = 0; b < 4; b++)
        t1_tma3(dst + b * kT1Box, map, (int)(o.tx * 128 + 32 * b), (int)(o.by * 8), (int)(o.bz * 8), mbar);
}

// select element j (0..7) of a register row without dynamic indexing
template <typename T>
__device__ __forceinline__ T t1_pick(const T (&v)[8], uint32_t j) {
    T r = v[0];
#pragma unroll
    for (int k = 1; k < 8; k++) r = (j == (uint32_t)k) ? v[k] : r;
    return r;
}
template <typename T>
__device__ __forceinline__ void t1_put(T (&v)[8], uint32_t j, T x) {
#pragma unroll
    for (int k = 0; k < 8; k++)
        if (j == (uint32_t)k) v[k] = x;
}

__global__ void __launch_bounds__(kT1Threads, 1)
    k_quantize3d8_tma(const __grid_constant__ T1Params P, const __grid_constant__ CUtensorMap map) {
    const Q3Params &p = P.q;
    extern __shared__ __align__(1024) unsigned char t1_smem[];
    // [stages x 16 KB tiles][s_col: warps x 16 bins x 32 lanes u32][s_codes: warps x 512 u16][s_hist: cap u32]
    __shared__ __align__(8) uint64_t s_full[kT1Stages];
    // per stage and warp: outlier count | slow-path flag << 31
    __shared__ uint32_t s_cnt[kT1Stages][kT1Warps];
    __shared__ uint64_t s_rec[kT1Stages][kT1Warps][kT1Sub][2];
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    const uint32_t tiles_s = ((uint32_t)__cvta_generic_to_shared(t1_smem) + 1023u) & ~1023u;
    unsigned char *tiles = t1_smem + (tiles_s - (uint32_t)__cvta_generic_to_shared(t1_smem));
    uint32_t *s_col = reinterpret_cast<uint32_t *>(tiles + kT1Stages * kT1Tile);
    uint16_t *s_codes = reinterpret_cast<uint16_t *>(s_col + kT1Warps * 16 * 32) + warp * 512;
    uint32_t *s_hist = s_col + kT1Warps * 16 * 32 + kT1Warps * 256;
    for (uint32_t i = threadIdx.x; i < kT1Warps * 16 * 32; i += blockDim.x) s_col[i] = 0;
    for (uint32_t i = threadIdx.x; i < p.cap; i += blockDim.x) s_hist[i] = 0;
    const uint32_t full_s = (uint32_t)__cvta_generic_to_shared(s_full);
    const uint64_t G = gridDim.x;
    T1Pos pos = t1_pos(P, blockIdx.x);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kT1Stages; s++) t1_mbar_init(full_s + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        T1Pos q = pos;
        for (int s = 0; s < kT1Stages; s++) {
            if (blockIdx.x + s * G < P.nst) t1_issue(&map, q, tiles_s + s * kT1Tile, full_s + 8 * s);
            t1_step(P, q);
        }
    }
    __syncthreads();
    const uint32_t hbase = (uint32_t)__cvta_generic_to_shared(s_hist);
    const uint32_t colbase = p.cap >= 16
        ? (uint32_t)__cvta_generic_to_shared(s_col + warp * 16 * 32) + lane * 4
        : 0xFFFFFFFFu;
    const uint32_t ly = lane & 7, lz0 = (lane >> 3) * 2;
    const uint64_t plane = p.g.nx * p.g.ny;
    const uint64_t lane_off = p.g.nx * ly + plane * lz0;
    const int32_t r = p.r;
    const uint32_t klo = p.cap >= 16 ? (uint32_t)(r - 8) : (uint32_t)(r + 16);
    const uint32_t sw = ly;  // SWIZZLE_128B: row R's 16-byte units are XORed with R & 7 (= ly here)
    const uint32_t R0 = ly + 8 * lz0, R1 = R0 + 8;
    const uint32_t j2 = (warp & 3) * 2;  // this warp's chunk = chunk (warp & 3) of box (warp >> 2)
    const uint32_t off00 = (warp >> 2) * kT1Box + R0 * 128 + ((j2 ^ sw) << 4);
    const uint32_t off01 = (warp >> 2) * kT1Box + R0 * 128 + (((j2 + 1) ^ sw) << 4);
    const uint32_t off10 = (warp >> 2) * kT1Box + R1 * 128 + ((j2 ^ sw) << 4);
    const uint32_t off11 = (warp >> 2) * kT1Box + R1 * 128 + (((j2 + 1) ^ sw) << 4);
    int flags = 0;
    uint32_t it = 0;
    for (uint64_t t = blockIdx.x; t < P.nst; t += G, it++, t1_step(P, pos)) {
        const uint32_t st = it % kT1Stages;
        const uint32_t bx = pos.tx * 16 + warp;
        const bool fast = ((uint64_t)pos.tx * 128 + 128 <= p.g.nx) && ((uint64_t)pos.by * 8 + 8 <= p.g.ny) &&
                          ((uint64_t)pos.bz * 8 + 8 <= p.g.nz);
        const uint64_t gi0 = (uint64_t)bx * 8 + p.g.nx * ((uint64_t)pos.by * 8) + plane * ((uint64_t)pos.bz * 8) +
                             lane_off;
        bool slow = !fast;
        uint32_t nout = 0;
        t1_mbar_wait(full_s + 8 * st, (it / kT1Stages) & 1u);
        if (fast) {
            float x0[8], x1[8];
            {
                const uint32_t bb = tiles_s + st * kT1Tile;
                float4 a, b2, c2, d;
                asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w)
                             : "r"(bb + off00));
                asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(b2.x), "=f"(b2.y), "=f"(b2.z), "=f"(b2.w)
                             : "r"(bb + off01));
                asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(c2.x), "=f"(c2.y), "=f"(c2.z), "=f"(c2.w)
                             : "r"(bb + off10));
                asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(d.x), "=f"(d.y), "=f"(d.z), "=f"(d.w)
                             : "r"(bb + off11));
                x0[0] = a.x; x0[1] = a.y; x0[2] = a.z; x0[3] = a.w;
                x0[4] = b2.x; x0[5] = b2.y; x0[6] = b2.z; x0[7] = b2.w;
                x1[0] = c2.x; x1[1] = c2.y; x1[2] = c2.z; x1[3] = c2.w;
                x1[4] = d.x; x1[5] = d.y; x1[6] = d.z; x1[7] = d.w;
            }
            int32_t d0[8], d1[8];
            bool ok = true;
            float kmax = 0.0f;
            // biased integers (f3::pq_fast_f32b): the deltas cancel the bias
            // everywhere but at the chunk origin, corrected after them
#pragma unroll
            for (int j = 0; j < 8; j++) {
                d0[j] = f3::pq_fast_f32b(x0[j], p.inv_hi, p.inv_lo, ok, kmax);
                d1[j] = f3::pq_fast_f32b(x1[j], p.inv_hi, p.inv_lo, ok, kmax);
            }
            const bool big = !(kmax < 4194304.0f);  // |k| >= 2^22 (or an infinity)
            if (!__all_sync(f3::kFull, ok && !big)) {
                // rare: an element near a rounding tie (exact f64 division for
                // it), or values beyond the int32 fast path (exact chunk path)
                if (__any_sync(f3::kFull, big)) {
                    slow = true;
                } else if (!ok) {
#pragma unroll 1
                    for (uint32_t b = 0; b < 16; b++) {
                        const uint32_t j = b & 7;
                        const float xv = b < 8 ? t1_pick(x0, j) : t1_pick(x1, j);
                        bool e = true;
                        float km = 0.0f;
                        (void)f3::pq_fast_f32b(xv, p.inv_hi, p.inv_lo, e, km);
                        if (!e) {
                            int fl = 0;
                            const int32_t v =
                                (int32_t)f3::pq_exact((double)xv, p.two_eb, p.slack, fl) + f3::kPqBias;
                            flags |= fl;
                            if (b < 8) t1_put(d0, j, v);
                            else t1_put(d1, j, v);
                        }
                    }
                }
            }
            if (!slow) {
                f3::deltas<int32_t>(d0, d1, lane);
                d0[0] -= lane == 0 ? f3::kPqBias : 0;
                uint32_t c0[8], c1[8];
                uint32_t o0 = 0, o1 = 0;
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    const bool i0 = (uint32_t)(d0[j] + r - 1) < (uint32_t)(2 * r - 1);  // |d| < r
                    const bool i1 = (uint32_t)(d1[j] + r - 1) < (uint32_t)(2 * r - 1);
                    c0[j] = i0 ? (uint32_t)(d0[j] + r) : (uint32_t)r;
                    c1[j] = i1 ? (uint32_t)(d1[j] + r) : (uint32_t)r;
                    o0 |= (uint32_t)!i0 << j;
                    o1 |= (uint32_t)!i1 << j;
                }
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
                const uint64_t sbase = plane * 8 * pos.bz + p.g.nx * 64 * pos.by + 512 * (uint64_t)bx;
                uint16_t *outp = static_cast<uint16_t *>(p.codes) + sbase;
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const uint32_t(&cr)[8] = h ? c1 : c0;
                    uint4 v;
                    v.x = cr[0] | (cr[1] << 16);
                    v.y = cr[2] | (cr[3] << 16);
                    v.z = cr[4] | (cr[5] << 16);
                    v.w = cr[6] | (cr[7] << 16);
                    *reinterpret_cast<uint4 *>(outp + 8 * (ly + 8 * (lz0 + h))) = v;
                }
                // outliers, ranked in stream order; the first kT1Sub go to the stage's record slots
                const uint32_t anym = __ballot_sync(f3::kFull, (o0 | o1) != 0);
                if (anym) {
                    const bool origin_only = anym == 1u && __shfl_sync(f3::kFull, (o0 == 1u && o1 == 0u) ? 1 : 0, 0);
                    if (origin_only) {
                        nout = 1;
                        if (lane == 0) {
                            s_rec[st][warp][0][0] = gi0;
                            s_rec[st][warp][0][1] = (uint64_t)(int64_t)d0[0];
                        }
                    } else {
                        uint32_t rk0, rk1;
                        f3::row_ranks(__popc(o0), __popc(o1), lane, rk0, rk1, nout);
#pragma unroll
                        for (int h = 0; h < 2; h++) {
                            uint32_t m = h ? o1 : o0, rk = h ? rk1 : rk0;
                            while (m) {
                                const uint32_t j = __ffs(m) - 1;
                                m &= m - 1;
                                if (rk < (uint32_t)kT1Sub) {
                                    s_rec[st][warp][rk][0] = gi0 + (h ? plane : 0) + j;
                                    s_rec[st][warp][rk][1] = (uint64_t)(int64_t)(h ? t1_pick(d1, j) : t1_pick(d0, j));
                                }
                                rk++;
                            }
                        }
                    }
                }
            }
        }
        if (slow) {
            // generic path (global reads, exact where needed); the tile's
            // records are re-derived in order by k_q3_emit (over_list)
            const uint64_t c = t * kT1Warps + warp;
            nout = 0;
            if (c < p.nchunks) {
                const Q3Res rr = q3_chunk_slow<float, uint16_t>(&p, c, lane, s_codes, nullptr, (uint32_t)kQ3Stash,
                                                                 s_hist);
                flags |= rr.flags;
                nout = rr.n;
            }
        }
        // release the stage: the tile's publisher warp (it mod 16, so every
        // warp publishes one tile in 16) waits on the stage's named barrier
        // for the other 15 (bar.arrive, non-blocking), publishes the two
        // outlier tiles and issues the stage's TMA refill.  The refill is what
        // the other warps wait for before they reuse the stage's slots, so
        // successive uses of a barrier cannot overlap.
        __syncwarp();
        if (lane == 0) s_cnt[st][warp] = nout | (slow ? 0x80000000u : 0u);
        const uint32_t pub = it % kT1Warps;
        if (warp != pub) {
            asm volatile("bar.arrive %0, %1;" ::"r"(1 + st), "r"(kT1Threads) : "memory");
        } else {
            asm volatile("bar.sync %0, %1;" ::"r"(1 + st), "r"(kT1Threads) : "memory");
            // two outlier tiles of 8 chunks: lanes 0-7 and 8-15
            const uint32_t sv = lane < kT1Warps ? s_cnt[st][lane] : 0u;
            const uint32_t cl = sv & 0x7FFFFFFFu;
            uint32_t inc = cl;
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) {
                const uint32_t v = __shfl_up_sync(f3::kFull, inc, o);
                if ((lane & 7) >= (uint32_t)o) inc += v;
            }
            const uint32_t tot0 = __shfl_sync(f3::kFull, inc, 7), tot1 = __shfl_sync(f3::kFull, inc, 15);
            const bool slow_st = __any_sync(f3::kFull, (sv >> 31) != 0);
            const uint32_t big = __ballot_sync(f3::kFull, lane < kT1Warps && cl > (uint32_t)kT1Sub);
            const bool over0 = slow_st || (big & 0xFFu), over1 = slow_st || (big & 0xFF00u);
            const uint64_t tile = 2 * t + (lane >> 3);
            if (lane < kT1Warps && !((lane >> 3) ? over1 : over0)) {
                uint64_t *tslot = p.slots + tile * 2 * kQ3Slot + 2 * (inc - cl);
                for (uint32_t k = 0; k < cl; k++) {
                    tslot[2 * k] = s_rec[st][lane][k][0];
                    tslot[2 * k + 1] = s_rec[st][lane][k][1];
                }
            }
            __syncwarp();  // every lane's reads of the stage bookkeeping are done
            if (lane == 0) {
                p.tile_cnt[2 * t] = tot0;
                p.tile_cnt[2 * t + 1] = tot1;
                if (over0) p.over_list[atomicAdd(p.n_over, 1u)] = (uint32_t)(2 * t);
                if (over1) p.over_list[atomicAdd(p.n_over, 1u)] = (uint32_t)(2 * t + 1);
                const uint64_t tn = t + kT1Stages * G;
                if (tn < P.nst) {
                    T1Pos q = pos;
#pragma unroll 1
                    for (int s = 0; s < kT1Stages; s++) t1_step(P, q);
                    t1_issue(&map, q, tiles_s + st * kT1Tile, full_s + 8 * st);
                }
            }
            __syncwarp();
        }
    }
    __syncwarp();
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
    flags = __reduce_or_sync(f3::kFull, flags);
    if (lane == 0 && flags) set_status(p.st, (flags & 1) ? LZB_E_OVERFLOW : LZB_E_ASSERT);
}

}  // namespace lzb
