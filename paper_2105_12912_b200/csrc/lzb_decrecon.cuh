// Fused K5 + K6 for ChunkSpec(8,8,8) grids of whole chunks, f32 output:
// decode a tile of 16 chunks (8192 symbols) of the Huffman stream straight
// into shared memory (K5 v4 tile decoder, lzb_dec4.cuh) and reconstruct the
// tile's chunks from there (outlier fuse + x/y/z partial sums + f64 dequant +
// min/max, TMA tensor stores), so the code stream never touches HBM.
// Included by lzb_recon.cu.  Reference: P/pipeline.py:318-326 (decompress) =
// P/huffman.py:64-122 (decode) + P/pipeline.py:108-117 (scatter) +
// P/reconstruct.py:22-88 (fuse, partial sums, dequantize).
//
// CTA = 4 decode warps + 8 reconstruct warps, persistent over tiles, two
// code tiles in shared memory.  Decode warps: stage the tile's stream words
// (cp.async), then thread per microblock (the plan from passes M/S gives each
// one's entry, count and first symbol) write the tile's symbols.  Reconstruct
// warps: warp w takes chunks w and w + 8 of the tile in the K6 register
// layout (lzb_fast3d.cuh).  Named barriers hand the tiles over, so decoding
// tile i+1 overlaps reconstructing tile i.
#pragma once

#include "lzb_dec4.cuh"
#include "lzb_recon3d.cuh"

namespace lzb {

constexpr uint32_t kFChunks = kD4Tile / 512;  // 8
constexpr uint32_t kFTileShift = 3;           // outlier buckets: 8-chunk tiles (as K6)

struct FParams {
    D4Plan d;
    R3Params r;
    int dbg;  // profiling only: 1 = decode without reconstructing, 2 = reconstruct without decoding  // r.codes unused; r.tile_start / r.brec bucket outliers per 16-chunk tile
};

// One chunk from the shared code tile (cs = its 512 u16 codes, chunk-major
// rows of 8), then dequantised into the warp's TMA tile buffer.
template <typename I>
__device__ __forceinline__ void f_chunk(const R3Params &p, const uint16_t *cs, uint32_t k, uint64_t r0,
                                        uint64_t r1, uint32_t lane, float &vmin, float &vmax, bool &overflow,
                                        bool reg_out, uint32_t rkey, int32_t rd, uint32_t nrec,
                                        uint32_t ybuf_s) {
    const uint32_t ly = lane & 7, lz0 = (lane >> 3) * 2;
    I v0[8], v1[8];
#pragma unroll
    for (int h = 0; h < 2; h++) {
        I(&v)[8] = h ? v1 : v0;
        const uint4 a = *reinterpret_cast<const uint4 *>(cs + 8 * (ly + 8 * (lz0 + h)));
        const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
        for (int j = 0; j < 4; j++) {
            v[2 * j] = (I)(int32_t)(w[j] & 0xFFFFu) - p.r;
            v[2 * j + 1] = (I)(int32_t)(w[j] >> 16) - p.r;
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
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const I(&v)[8] = h ? v1 : v0;
        float o[8];
#pragma unroll
        for (int j = 0; j < 8; j++) {
            o[j] = (float)__dmul_rn((double)v[j], p.two_eb);
            vmin = fminf(vmin, o[j]);
            vmax = fmaxf(vmax, o[j]);
        }
        const uint32_t a = ybuf_s + (ly + 8 * (lz0 + h)) * 32;
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(o[0]), "f"(o[1]), "f"(o[2]),
                     "f"(o[3]));
        asm volatile("st.shared.v4.f32 [%0+16], {%1, %2, %3, %4};" ::"r"(a), "f"(o[4]), "f"(o[5]), "f"(o[6]),
                     "f"(o[7]));
    }
}

__device__ __noinline__ void f_chunk_wide(const R3Params *p, const uint16_t *cs, uint32_t k, uint64_t r0,
                                          uint64_t r1, uint32_t lane, float *mm, bool *ovf, uint32_t ybuf_s) {
    float vmin = mm[0], vmax = mm[1];
    bool o = *ovf;
    f_chunk<int64_t>(*p, cs, k, r0, r1, lane, vmin, vmax, o, false, 0, 0, 0, ybuf_s);
    mm[0] = vmin;
    mm[1] = vmax;
    *ovf = o;
}

// Named barriers (0 is __syncthreads): FULL[s] = 1 + s, EMPTY[s] = 3 + s,
// decode-warp-only = 5.
__device__ __forceinline__ void nbar_sync(uint32_t id, uint32_t n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void nbar_arrive(uint32_t id, uint32_t n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

constexpr int kFWarps = 8;
constexpr int kFThreads = 32 * kFWarps;
constexpr uint32_t kFRangeChunks = 32;                 // chunks per range (one decode + reconstruct round)
constexpr uint32_t kFRange = kFRangeChunks * 512;      // symbols per range
constexpr uint32_t kFStgW = 136;                       // staged words per subsequence
// dynamic shared memory: the range's code buffer, per warp two subsequence
// word stages and two TMA store tiles
// (+ the decode LUT: in shared memory, not L1, which the rest of the CTA's
// shared memory squeezes)
constexpr size_t kFSmem = (size_t)kFRange * 2 + (size_t)kFWarps * 2 * kFStgW * 4 + (size_t)kFWarps * 4096 +
                          (size_t)kLutSize * 8;

// A CTA takes ranges of 32 consecutive chunks.  Decode: warp per subsequence
// of the stream (lane per 128-bit microblock, all lanes busy; words staged by
// cp.async, the next subsequence in flight), every microblock's symbols land
// at their offset in the range's code buffer.  Reconstruct: warp w takes
// chunks w, w+8, w+16, w+24 (the K6 register layout), TMA stores.
__global__ void __launch_bounds__(kFThreads, 2)
    k_decrecon3d8(const __grid_constant__ FParams P, const __grid_constant__ CUtensorMap ymap) {
    extern __shared__ __align__(128) unsigned char f_smem[];
    __shared__ DecCanon s_can;
    uint16_t *buf = reinterpret_cast<uint16_t *>(f_smem);
    uint64_t *s_l8 = reinterpret_cast<uint64_t *>(f_smem + kFRange * 2 + kFWarps * 2 * kFStgW * 4 + kFWarps * 4096);
    for (uint32_t i = threadIdx.x; i < kLutSize; i += blockDim.x) s_l8[i] = P.d.tab->lut8[i];
    load_canon(s_can, P.d.tab);
    __syncthreads();
    if (P.d.st->code) return;  // the plan asked for the robust decoder (or the book is invalid)
    const D4Plan &d = P.d;
    const R3Params &p = P.r;
    const uint32_t b8 = (uint32_t)d.base8 & 0xFFFFu;
    const D4Luts L{d.tab->lut8, smem_addr(s_l8), b8 | (b8 << 16), d.tab->lut1, d.tab->lut1s, &s_can, d.syms};
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    const uint32_t wst_s = smem_addr(f_smem + kFRange * 2) + warp * 2 * kFStgW * 4;
    const uint32_t ybase_s = smem_addr(f_smem + kFRange * 2 + kFWarps * 2 * kFStgW * 4) + warp * 4096;
    const uint64_t nranges = (p.nchunks + kFRangeChunks - 1) / kFRangeChunks;
    float vmin = INFINITY, vmax = -INFINITY;
    uint32_t qmn = 0x7FFF7FFFu, qmx = 0x80008000u;  // packed int16 min / max of the 16-bit path's q
    const bool narrow = p.r <= 2048;                 // cap <= 4096: |q'| of a code < 2^11
    bool overflow = false;
    uint32_t nb = 0;  // TMA stores issued by this warp
    const uint32_t nbx = (uint32_t)p.g.nbx, nby = (uint32_t)p.g.nby;
    for (uint64_t rg = blockIdx.x; rg < nranges; rg += gridDim.x) {
        const uint64_t A = rg * kFRange;
        const uint64_t ta = rg * (kFRange / kD4Tile), tb = umin64(ta + kFRange / kD4Tile, d.ntiles);
        const uint64_t ma = d.tfirst[ta], mb = d.tfirst[tb];
        const uint64_t s0 = ma / 32, s1 = mb / 32;
        __syncthreads();  // every warp is done reconstructing the previous range
        // ---- decode: warp per subsequence ----
        if (P.dbg < 2) {
            uint64_t sq = s0 + warp;
            uint32_t sb = 0;
            if (sq <= s1) d4_stage_words(d, sq * 128, kFStgW, wst_s, lane, 32);
            asm volatile("cp.async.commit_group;" ::: "memory");
            for (; sq <= s1; sq += kFWarps, sb ^= 1) {
                const uint64_t nx = sq + kFWarps;
                if (nx <= s1) d4_stage_words(d, nx * 128, kFStgW, wst_s + (sb ^ 1) * kFStgW * 4, lane, 32);
                asm volatile("cp.async.commit_group;" ::: "memory");
                const uint64_t m = sq * 32 + lane;
                const bool in = m >= ma && m <= mb;
                const uint32_t cpv = in ? d.cp[m] : 0u;
                const uint64_t o = in ? d.mboff[m] : 0ull;
                asm volatile("cp.async.wait_group 1;" ::: "memory");
                __syncwarp();
                const uint32_t c = cpv >> 8;
                if (in && c && o + c > A && o < A + kFRange) {
                    SRd r;
                    r.init(wst_s + sb * kFStgW * 4, lane * kD4MB + d.head + (cpv & 0xFFu));
                    d4_tile_decode_rd<kFRange>(r, L, (int32_t)((int64_t)o - (int64_t)A),
                                               (uint32_t)umin64(c, A + kFRange - o), buf);
                }
                __syncwarp();  // the lanes are done with this word stage
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
        }
        __syncthreads();  // the range's codes are complete
        if (P.dbg == 1) continue;
        // ---- reconstruct ----
#pragma unroll 1
        for (uint32_t kk = warp; kk < kFRangeChunks; kk += kFWarps) {
            const uint64_t cg = rg * kFRangeChunks + kk;
            if (cg >= p.nchunks) break;
            const uint64_t tt = cg >> 3;  // the K6 outlier tile (8 chunks)
            const uint32_t k = (uint32_t)(cg & 7);
            const uint64_t r0 = p.tile_start[tt], r1 = p.tile_start[tt + 1];
            const uint64_t nr64 = r1 - r0;
            const bool reg_out = nr64 <= 32;
            const uint32_t nrec = reg_out ? (uint32_t)nr64 : 0u;
            uint32_t rkey = 0xFFFFFFFFu;
            int32_t rd = 0;
            bool wide_l = false;
            if (reg_out && lane < nrec) {
                rkey = (uint32_t)p.brec[2 * (r0 + lane)];
                const int64_t dl = (int64_t)p.brec[2 * (r0 + lane) + 1];
                wide_l = (rkey >> 9) == k && (dl >= (1ll << 20) || dl <= -(1ll << 20));
                rd = (int32_t)dl;
            }
            const uint32_t c32 = (uint32_t)cg;  // < 2^32 chunks (host checks)
            const uint32_t byz = c32 / nbx, bx = c32 - byz * nbx, by = byz % nby, bz = byz / nby;
            const uint16_t *cs = buf + kk * 512;
            const uint32_t yb = ybase_s + (nb & 1u) * 2048;
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncwarp();
            const bool wide = __any_sync(f3::kFull, reg_out ? wide_l : (r1 > r0 && r3_needs_wide(p, r0, r1, k)));
            if (wide) {
                float mmv[2] = {vmin, vmax};
                f_chunk_wide(&p, cs, k, r0, r1, lane, mmv, &overflow, yb);
                vmin = mmv[0];
                vmax = mmv[1];
            } else if (!(narrow && reg_out &&
                         r3_chunk16(p, *reinterpret_cast<const uint4 *>(cs + 8 * ((lane & 7) + 16 * (lane >> 3))),
                                    *reinterpret_cast<const uint4 *>(cs + 8 * ((lane & 7) + 16 * (lane >> 3) + 8)), k,
                                    lane, qmn, qmx, rkey, rd, nrec, yb))) {
                f_chunk<int32_t>(p, cs, k, r0, r1, lane, vmin, vmax, overflow, reg_out, rkey, rd, nrec, yb);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0 && P.dbg != 3) r3_tma_store(&ymap, yb, bx * 8, by * 8, bz * 8);
            nb++;
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    {  // the 16-bit path's extremes: the dequantisation is monotone in q
        const int32_t lo = min(v2lo(qmn), v2hi(qmn)), hi = max(v2lo(qmx), v2hi(qmx));
        if (lo <= hi) {
            vmin = fminf(vmin, (float)__dmul_rn((double)lo, p.two_eb));
            vmax = fmaxf(vmax, (float)__dmul_rn((double)hi, p.two_eb));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        vmin = fminf(vmin, __shfl_xor_sync(f3::kFull, vmin, o));
        vmax = fmaxf(vmax, __shfl_xor_sync(f3::kFull, vmax, o));
    }
    if (lane == 0 && vmin <= vmax) {
        atomicMin(&p.mm[0], r3_dkey((double)vmin));
        atomicMax(&p.mm[1], r3_dkey((double)vmax));
    }
    if (__any_sync(f3::kFull, overflow) && lane == 0) set_status(p.st, LZB_E_OVERFLOW);
}

}  // namespace lzb
