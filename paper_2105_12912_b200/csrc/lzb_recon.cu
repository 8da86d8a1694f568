// K6: fused outlier fuse + chunk-wise multi-dimensional partial-sum
// reconstruction + dequantization + range / finiteness, plus the stand-alone
// field range and quality-statistics kernels.
//
// Reference semantics (P = /root/reference/pkg/src/lzebc):
//   scatter_chunk_major  P/pipeline.py:108-117
//   _decode_outliers     P/pipeline.py:306-315  (index < count, strictly increasing)
//   fuse_outliers        P/reconstruct.py:22-32 q' = code - r, q'[idx] += delta (ADD)
//   reconstruct_chunk    P/reconstruct.py:40-57 f64 sum |q'| >= 2^62 -> overflow;
//                        inclusive prefix sums along x, y, z inside each chunk
//   dequantize           P/reconstruct.py:79-88 f64(q) * (2 eb) -> dtype; finite
//   Field range          P/grid.py:155-202
//   stats                P/pipeline.py:329-345
//
// Design (K6): the same tiles as K1 (K whole chunks along x in one
// chunk row).  The tile's contiguous chunk-major code range is read
// coalesced into shared memory as int64 q' (box layout), the tile's outliers
// (bucketed per tile by a counting sort) are added, then prefix sums run in
// shared memory: x as one segmented block scan over the box (segments = chunk
// x-lines), y and z as per-line sequential scans.  Dequantised values are
// written in grid order (coalesced along x) with a fused min/max/finite
// reduction.  Prefix sums along different axes commute, so the order of the
// three passes does not matter for the (exact integer) result.
#include <string.h>

#include "lzb_common.cuh"
#include "lzb_recon3d.cuh"
#include "lzb_recon2d.cuh"

namespace lzb {

// Reduction slots {min key, max key, first bad offset, 0}: set by a kernel,
// not a (pageable) host copy, so it never waits on a copy engine.
__global__ void k_mm_init(unsigned long long *mm, int n) {
    if (threadIdx.x < (unsigned)n) mm[threadIdx.x] = (threadIdx.x & 1) ? 0ull : ~0ull;
}

constexpr int kRcThreads = 256;
constexpr int kRcTile = 4096;
constexpr int kRcItems = kRcTile / kRcThreads;  // 16
constexpr double kPsumLimit = 4611686018427387904.0;  // 2^62, P/reconstruct.py:19

// order-preserving map of doubles to u64 (for atomic min/max)
__device__ __forceinline__ unsigned long long dkey(double v) {
    unsigned long long b = __double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dunkey(unsigned long long k) {
    unsigned long long b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
    return __longlong_as_double(b);
}

struct RcParams {
    const void *codes;
    Geom g;
    double two_eb;
    int64_t radius;
    uint32_t cap;
    void *y;
    int64_t *pre;  // optional prequant output (grid order)
    lzb_dstatus *st;
    unsigned long long *mm;  // [min key, max key, first bad offset]
    // tiles (same as K1 box mode)
    uint32_t K;
    uint64_t tiles_per_row;
    uint64_t ntiles;
    // outliers bucketed per tile: (box-local position u32 | pad, delta i64)
    const uint64_t *tile_start;  // ntiles + 1
    const uint64_t *brec;        // 2 u64 per record
};

struct RTile {
    uint64_t X0, Y0, Z0;
    uint32_t BX, EY, EZ, kc, cx, last_ex;
    uint64_t base;
    uint32_t n;
};

__device__ __forceinline__ RTile rtile(const Geom &g, uint32_t K, uint64_t tiles_per_row, uint64_t t) {
    uint64_t row = t / tiles_per_row, j = t - row * tiles_per_row;
    uint64_t bx0 = j * K, by = row % g.nby, bz = row / g.nby;
    RTile b;
    b.kc = (uint32_t)umin64(K, g.nbx - bx0);
    b.X0 = bx0 * g.cx;
    b.Y0 = by * g.cy;
    b.Z0 = bz * g.cz;
    b.BX = (uint32_t)umin64((uint64_t)b.kc * g.cx, g.nx - b.X0);
    b.EY = (uint32_t)umin64(g.cy, g.ny - b.Y0);
    b.EZ = (uint32_t)umin64(g.cz, g.nz - b.Z0);
    b.cx = (uint32_t)g.cx;
    b.last_ex = b.BX - (b.kc - 1) * b.cx;
    b.base = chunk_base(g, bx0, by, bz);
    b.n = b.BX * b.EY * b.EZ;
    return b;
}

// stream position in tile -> box index
__device__ __forceinline__ uint32_t rt_box_index(const RTile &b, uint32_t p) {
    uint32_t full = b.cx * b.EY * b.EZ;
    uint32_t k = p / full;
    uint32_t r = p - k * full;
    uint32_t ex = (k == b.kc - 1) ? b.last_ex : b.cx;
    uint32_t exy = ex * b.EY;
    uint32_t lz = r / exy;
    r -= lz * exy;
    uint32_t ly = r / ex;
    uint32_t lx = r - ly * ex;
    return (k * b.cx + lx) + b.BX * (ly + b.EY * lz);
}

template <typename SymT, typename OutT>
__global__ void __launch_bounds__(kRcThreads, 4) k_reconstruct(RcParams p) {
    __shared__ int64_t s_q[kRcTile];
    __shared__ int64_t s_cv[32];
    __shared__ uint32_t s_cf[32];
    __shared__ double s_sum[64];
    __shared__ int s_big;
    const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
    double vmin = INFINITY, vmax = -INFINITY;
    unsigned long long bad = ~0ull;
    bool overflow = false;
    const bool line = p.g.ny == 1 && p.g.nz == 1;  // 1D geometry: no index divisions
    const bool cx_pow2 = (p.g.cx & (p.g.cx - 1)) == 0;
    for (uint64_t t = blockIdx.x; t < p.ntiles; t += gridDim.x) {
        const RTile b = rtile(p.g, p.K, p.tiles_per_row, t);
        const SymT *cs = static_cast<const SymT *>(p.codes) + b.base;
        if (tid == 0) s_big = 0;
        // ---- codes -> q' (box layout) ----
        for (uint32_t i = tid; i < b.n; i += kRcThreads)
            s_q[line ? i : rt_box_index(b, i)] = (int64_t)cs[i] - p.radius;
        __syncthreads();
        // ---- fuse this tile's outliers (unique positions: plain adds) ----
        const uint64_t r0 = p.tile_start[t], r1 = p.tile_start[t + 1];
        for (uint64_t k = r0 + tid; k < r1; k += kRcThreads)
            s_q[(uint32_t)p.brec[2 * k]] += (int64_t)p.brec[2 * k + 1];
        __syncthreads();
        // ---- overflow guard (P/reconstruct.py:48-53): only chunks holding a
        // |q'| >= 2^50 can reach 2^62 (chunk volume <= 4096) ----
        {
            int big = 0;
            for (uint32_t i = tid; i < b.n; i += kRcThreads) {
                int64_t v = s_q[i];
                if (v >= (1ll << 50) || v <= -(1ll << 50)) big = 1;
            }
            if (__any_sync(0xffffffffu, big) && lane == 0) s_big = 1;
            __syncthreads();
            if (s_big) {
                // per chunk, sequential f64 sum in row-major chunk order (thread per chunk)
                for (uint32_t k = tid; k < b.kc; k += kRcThreads) {
                    uint32_t ex = (k == b.kc - 1) ? b.last_ex : b.cx;
                    double tot = 0.0;
                    for (uint32_t z = 0; z < b.EZ; z++)
                        for (uint32_t y = 0; y < b.EY; y++)
                            for (uint32_t x = 0; x < ex; x++) {
                                int64_t v = s_q[(k * b.cx + x) + b.BX * (y + b.EY * z)];
                                tot += fabs((double)v);
                            }
                    if (tot >= kPsumLimit) overflow = true;
                }
                __syncthreads();
            }
        }
        // ---- x: segmented block scan over the box; heads at chunk x-line starts ----
        {
            const uint32_t i0 = tid * kRcItems;
            int64_t v[kRcItems];
            uint32_t flags = 0;
            int64_t run = 0;
            // 1D: position inside the chunk, advanced without divisions
            uint32_t mx = line ? (cx_pow2 ? (i0 & (b.cx - 1)) : i0 % b.cx) : 0u;
#pragma unroll
            for (int k = 0; k < kRcItems; k++) {
                uint32_t i = i0 + k;
                bool head = false;
                if (i < b.n) {
                    if (line) {
                        head = mx == 0;
                        mx = mx + 1 == b.cx ? 0u : mx + 1;
                    } else {
                        uint32_t bxl = i % b.BX;
                        head = (bxl % b.cx) == 0;
                    }
                    int64_t q = s_q[i];
                    run = head ? q : run + q;
                    v[k] = run;
                } else {
                    v[k] = 0;
                    head = true;
                    run = 0;
                }
                flags |= (uint32_t)head << k;
            }
            // (flag, value) segmented inclusive scan of thread aggregates
            uint32_t f = flags != 0;
            int64_t agg = run;  // value since the last head (or whole range)
            // inclusive warp scan
            int64_t sv = agg;
            uint32_t sf = f;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int64_t pv = __shfl_up_sync(0xffffffffu, sv, o);
                uint32_t pf = __shfl_up_sync(0xffffffffu, sf, o);
                if (lane >= (uint32_t)o) {
                    if (!sf) sv += pv;
                    sf |= pf;
                }
            }
            if (lane == 31) {
                s_cv[warp] = sv;
                s_cf[warp] = sf;
            }
            __syncthreads();
            if (warp == 0) {
                // inclusive scan of the warp aggregates; identity is (flag 0, value 0)
                int64_t wv = lane < (kRcThreads / 32) ? s_cv[lane] : 0;
                uint32_t wf = lane < (kRcThreads / 32) ? s_cf[lane] : 0;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    int64_t pv = __shfl_up_sync(0xffffffffu, wv, o);
                    uint32_t pf = __shfl_up_sync(0xffffffffu, wf, o);
                    if (lane >= (uint32_t)o) {
                        if (!wf) wv += pv;
                        wf |= pf;
                    }
                }
                if (lane < (kRcThreads / 32)) {
                    s_cv[lane] = wv;
                    s_cf[lane] = wf;
                }
            }
            __syncthreads();
            // exclusive prefix of this thread = (warps before) (+) (lanes before)
            int64_t ev = __shfl_up_sync(0xffffffffu, sv, 1);
            uint32_t ef = __shfl_up_sync(0xffffffffu, sf, 1);
            if (lane == 0) {
                ev = 0;
                ef = 0;
            }
            const int64_t wprev = warp > 0 ? s_cv[warp - 1] : 0;
            const int64_t cv = ef ? ev : wprev + ev;
            // apply carry up to the first head in this thread's range
#pragma unroll
            for (int k = 0; k < kRcItems; k++) {
                if ((flags >> k) & 1u) break;
                v[k] += cv;
            }
#pragma unroll
            for (int k = 0; k < kRcItems; k++)
                if (i0 + k < b.n) s_q[i0 + k] = v[k];
        }
        __syncthreads();
        // ---- y: per (x, z) column ----
        if (b.EY > 1)
            for (uint32_t c = tid; c < b.BX * b.EZ; c += kRcThreads) {
                uint32_t x = c % b.BX, z = c / b.BX;
                uint32_t i = x + b.BX * b.EY * z;
                int64_t acc = s_q[i];
                for (uint32_t yy = 1; yy < b.EY; yy++) {
                    i += b.BX;
                    acc += s_q[i];
                    s_q[i] = acc;
                }
            }
        __syncthreads();
        // ---- z: per (x, y) pillar ----
        if (b.EZ > 1)
            for (uint32_t c = tid; c < b.BX * b.EY; c += kRcThreads) {
                uint32_t i = c;
                int64_t acc = s_q[i];
                for (uint32_t zz = 1; zz < b.EZ; zz++) {
                    i += b.BX * b.EY;
                    acc += s_q[i];
                    s_q[i] = acc;
                }
            }
        __syncthreads();
        // ---- dequantize, range, write grid order ----
        const uint32_t bxy = b.BX * b.EY;
        OutT *yo = static_cast<OutT *>(p.y);
        for (uint32_t i = tid; i < b.n; i += kRcThreads) {
            uint64_t gi;
            if (line) {
                gi = b.X0 + i;
            } else {
                uint32_t z = i / bxy, rem = i - z * bxy, yy = rem / b.BX, x = rem - yy * b.BX;
                gi = (b.X0 + x) + p.g.nx * ((b.Y0 + yy) + p.g.ny * (b.Z0 + z));
            }
            int64_t q = s_q[i];
            double d = __dmul_rn((double)q, p.two_eb);
            OutT o = (OutT)d;
            yo[gi] = o;
            if (p.pre) p.pre[gi] = q;
            double od = (double)o;
            if (!isfinite(od)) {
                if (gi < bad) bad = gi;
            } else {
                vmin = fmin(vmin, od);
                vmax = fmax(vmax, od);
            }
        }
        __syncthreads();
    }
    // block reduce min/max/bad via warp ops then global atomics
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        vmin = fmin(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
        vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
        unsigned long long ob = __shfl_xor_sync(0xffffffffu, bad, o);
        bad = ob < bad ? ob : bad;
    }
    if (lane == 0) {
        if (vmin <= vmax) {
            atomicMin(&p.mm[0], dkey(vmin));
            atomicMax(&p.mm[1], dkey(vmax));
        }
        if (bad != ~0ull) atomicMin(&p.mm[2], bad);
    }
    if (__any_sync(0xffffffffu, overflow) && lane == 0) set_status(p.st, LZB_E_OVERFLOW);
    (void)s_sum;
}

// ---- outlier validation + per-tile bucketing ----
struct OutParams {
    const uint8_t *rec;  // 16-byte LE records, any alignment
    uint64_t n_out;
    int fast3d;          // tiles = 2^tshift consecutive chunk ordinals (8: K6, 16: fused K5+K6)
    int fast2d;          // ChunkSpec(16,16): tiles of 8 chunk ordinals, key k << 8 | y << 4 | x
    int fast1d;          // ChunkSpec(256) 1D: tiles of 8 chunks, key k << 8 | x mod 256
    uint32_t tshift;
    Geom g;
    uint32_t K;
    uint64_t tiles_per_row;
    uint64_t ntiles;
    uint32_t *tile_cnt;
    uint32_t *tile_fill;
    uint64_t *tile_start;
    uint64_t *brec;
    lzb_dstatus *st;
};

__device__ __forceinline__ uint64_t ld_le64(const uint8_t *p) {
    uint64_t v = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) v |= (uint64_t)p[k] << (8 * k);
    return v;
}

// tile id + box-local position of a global index
__device__ __forceinline__ uint64_t tile_of(const OutParams &p, uint64_t idx, uint32_t *boxpos) {
    const Geom &g = p.g;
    uint64_t x = idx % g.nx, yz = idx / g.nx;
    uint64_t y = yz % g.ny, z = yz / g.ny;
    uint64_t bx = x / g.cx, by = y / g.cy, bz = z / g.cz;
    if (p.fast1d) {
        *boxpos = (uint32_t)((((x >> 8) & 7u) << 8) | (x & 255));
        return x >> 11;
    }
    if (p.fast2d) {
        const uint64_t ord = bx + g.nbx * by;
        *boxpos = (uint32_t)(((ord & 7u) << 8) | ((y & 15) << 4) | (x & 15));
        return ord >> 3;
    }
    if (p.fast3d) {
        uint64_t ord = bx + g.nbx * (by + g.nby * bz);
        *boxpos = (uint32_t)(((ord & ((1u << p.tshift) - 1u)) << 9) | ((z & 7) << 6) | ((y & 7) << 3) | (x & 7));
        return ord >> p.tshift;
    }
    uint64_t j = bx / p.K;
    uint64_t t = (bz * g.nby + by) * p.tiles_per_row + j;
    uint64_t X0 = j * p.K * g.cx;
    uint32_t BX = (uint32_t)umin64((uint64_t)umin64(p.K, g.nbx - j * p.K) * g.cx, g.nx - X0);
    uint32_t EY = (uint32_t)umin64(g.cy, g.ny - by * g.cy);
    *boxpos = (uint32_t)(x - X0) + BX * ((uint32_t)(y - by * g.cy) + EY * (uint32_t)(z - bz * g.cz));
    return t;
}

__global__ void k_out_count(OutParams p) {
    int bad = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < p.n_out;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t idx = ld_le64(p.rec + 16 * i);
        uint64_t total = p.g.nx * p.g.ny * p.g.nz;
        if (idx >= total) {
            bad = 1;
            continue;
        }
        if (i > 0 && !(ld_le64(p.rec + 16 * (i - 1)) < idx)) bad = 1;
        uint32_t bp;
        uint64_t t = tile_of(p, idx, &bp);
        atomicAdd(&p.tile_cnt[t], 1u);
    }
    if (__any_sync(0xffffffffu, bad) && lane_id() == 0) set_status(p.st, LZB_E_CORRUPT);
}

__global__ void k_out_scatter(OutParams p) {
    if (p.st->code) return;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < p.n_out;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t idx = ld_le64(p.rec + 16 * i);
        uint32_t bp;
        uint64_t t = tile_of(p, idx, &bp);
        uint64_t slot = p.tile_start[t] + atomicAdd(&p.tile_fill[t], 1u);
        p.brec[2 * slot] = bp;
        p.brec[2 * slot + 1] = ld_le64(p.rec + 16 * i + 8);
    }
}

// exclusive scan u32 -> u64 (ntiles + 1 outputs), look-back
__global__ void __launch_bounds__(256) k_scan_tiles(const uint32_t *in, uint64_t *out, uint64_t n,
                                                    uint64_t *lb, unsigned int *ticket) {
    __shared__ uint64_t s_t, s_ex;
    __shared__ uint64_t s_scan[33];
    const uint64_t ntl = (n + 1 + 2047) / 2048;
    while (true) {
        if (threadIdx.x == 0) s_t = atomicAdd(ticket, 1u);
        __syncthreads();
        const uint64_t t = s_t;
        if (t >= ntl) break;
        const uint64_t base = t * 2048 + threadIdx.x * 8;
        uint64_t v[8], sum = 0;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            v[k] = base + k < n ? in[base + k] : 0;
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
            if (base + k <= n) out[base + k] = run;
            run += v[k];
        }
        __syncthreads();
    }
}

__global__ void k_rc_finish(lzb_dstatus *st, const unsigned long long *mm) {
    st->u[0] = __double_as_longlong(dunkey(mm[0]));
    st->u[1] = __double_as_longlong(dunkey(mm[1]));
    st->u[2] = mm[2];
    if (mm[2] != ~0ull) set_status(st, LZB_E_DATA);
}

// ---- generic fallback for chunks larger than a tile: global int64 passes ----
__global__ void k_gen_fuse(const void *codes, int code_bytes, Geom g, int64_t radius, int64_t *q) {
    const uint64_t n = g.nx * g.ny * g.nz;
    for (uint64_t pos = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; pos < n;
         pos += (uint64_t)gridDim.x * blockDim.x) {
        // stream position -> grid index (same decomposition as K1's stream mode)
        uint64_t layer = g.nx * g.ny * g.cz;
        uint64_t bz = pos / layer, r = pos - bz * layer;
        uint64_t ez = umin64(g.cz, g.nz - bz * g.cz);
        uint64_t rowsz = g.nx * ez * g.cy;
        uint64_t by = r / rowsz;
        r -= by * rowsz;
        uint64_t ey = umin64(g.cy, g.ny - by * g.cy);
        uint64_t csz = ez * ey * g.cx;
        uint64_t bx = r / csz;
        r -= bx * csz;
        uint64_t ex = umin64(g.cx, g.nx - bx * g.cx);
        uint64_t lz = r / (ex * ey);
        r -= lz * ex * ey;
        uint64_t ly = r / ex, lx = r - ly * ex;
        uint64_t gi = (bx * g.cx + lx) + g.nx * ((by * g.cy + ly) + g.ny * (bz * g.cz + lz));
        uint32_t c = code_bytes == 2 ? static_cast<const uint16_t *>(codes)[pos]
                                     : static_cast<const uint32_t *>(codes)[pos];
        q[gi] = (int64_t)c - radius;
    }
}

__global__ void k_gen_outliers(const uint8_t *rec, uint64_t n_out, uint64_t total, int64_t *q,
                               lzb_dstatus *st) {
    int bad = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_out;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t idx = ld_le64(rec + 16 * i);
        if (idx >= total || (i > 0 && !(ld_le64(rec + 16 * (i - 1)) < idx))) {
            bad = 1;
            continue;
        }
        q[idx] += (int64_t)ld_le64(rec + 16 * i + 8);
    }
    if (__any_sync(0xffffffffu, bad) && lane_id() == 0) set_status(st, LZB_E_CORRUPT);
}

// thread per chunk: overflow guard + x, y, z scans in global memory
__global__ void k_gen_psum(Geom g, int64_t *q, lzb_dstatus *st) {
    const uint64_t nch = g.nbx * g.nby * g.nbz;
    for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < nch;
         c += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t bx = c % g.nbx, by = (c / g.nbx) % g.nby, bz = c / (g.nbx * g.nby);
        uint64_t x0 = bx * g.cx, y0 = by * g.cy, z0 = bz * g.cz;
        uint64_t ex = umin64(g.cx, g.nx - x0), ey = umin64(g.cy, g.ny - y0), ez = umin64(g.cz, g.nz - z0);
        auto at = [&](uint64_t lx, uint64_t ly, uint64_t lz) -> int64_t & {
            return q[(x0 + lx) + g.nx * ((y0 + ly) + g.ny * (z0 + lz))];
        };
        double tot = 0.0;
        for (uint64_t lz = 0; lz < ez; lz++)
            for (uint64_t ly = 0; ly < ey; ly++)
                for (uint64_t lx = 0; lx < ex; lx++) tot += fabs((double)at(lx, ly, lz));
        if (tot >= kPsumLimit) {
            set_status(st, LZB_E_OVERFLOW);
            continue;
        }
        for (uint64_t lz = 0; lz < ez; lz++)
            for (uint64_t ly = 0; ly < ey; ly++)
                for (uint64_t lx = 1; lx < ex; lx++) at(lx, ly, lz) += at(lx - 1, ly, lz);
        for (uint64_t lz = 0; lz < ez; lz++)
            for (uint64_t ly = 1; ly < ey; ly++)
                for (uint64_t lx = 0; lx < ex; lx++) at(lx, ly, lz) += at(lx, ly - 1, lz);
        for (uint64_t lz = 1; lz < ez; lz++)
            for (uint64_t ly = 0; ly < ey; ly++)
                for (uint64_t lx = 0; lx < ex; lx++) at(lx, ly, lz) += at(lx, ly, lz - 1);
    }
}

template <typename OutT>
__global__ void k_gen_dequant(const int64_t *q, uint64_t n, double two_eb, OutT *y, int64_t *pre,
                              unsigned long long *mm) {
    double vmin = INFINITY, vmax = -INFINITY;
    unsigned long long bad = ~0ull;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        OutT o = (OutT)__dmul_rn((double)q[i], two_eb);
        y[i] = o;
        if (pre) pre[i] = q[i];
        double od = (double)o;
        if (!isfinite(od)) {
            if (i < bad) bad = i;
        } else {
            vmin = fmin(vmin, od);
            vmax = fmax(vmax, od);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        vmin = fmin(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
        vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
        unsigned long long ob = __shfl_xor_sync(0xffffffffu, bad, o);
        bad = ob < bad ? ob : bad;
    }
    if (lane_id() == 0) {
        if (vmin <= vmax) {
            atomicMin(&mm[0], dkey(vmin));
            atomicMax(&mm[1], dkey(vmax));
        }
        if (bad != ~0ull) atomicMin(&mm[2], bad);
    }
}

// ---- field range (P/grid.py:155-202) ----
// One streaming pass: 16-byte loads, four in flight per thread, min/max in the
// input precision (exact), the first non-finite offset by an atomic min.
template <typename InT>
__device__ __forceinline__ void fr_take(InT v, uint64_t i, InT &vmin, InT &vmax, unsigned long long &bad) {
    if (!isfinite(v)) {
        if (i < bad) bad = i;
    } else {
        vmin = v < vmin ? v : vmin;
        vmax = v > vmax ? v : vmax;
    }
}

template <typename InT>
__global__ void __launch_bounds__(256) k_field_range(const InT *x, uint64_t n, unsigned long long *mm) {
    constexpr int V = 16 / sizeof(InT);  // elements per 16-byte load
    constexpr int U = 4;                 // loads in flight per thread
    InT vmin = (InT)INFINITY, vmax = (InT)-INFINITY;
    unsigned long long bad = ~0ull;
    const bool aligned = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    const uint64_t nv = aligned ? n / V : 0;  // whole vectors
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
    const uint4 *xv = reinterpret_cast<const uint4 *>(x);
    uint64_t b = tid;
    for (; b + (U - 1) * nt < nv; b += U * nt) {
        uint4 w[U];
#pragma unroll
        for (int u = 0; u < U; u++) w[u] = __ldcs(xv + b + u * nt);
#pragma unroll
        for (int u = 0; u < U; u++) {
            const InT *e = reinterpret_cast<const InT *>(&w[u]);
#pragma unroll
            for (int k = 0; k < V; k++) fr_take<InT>(e[k], (b + u * nt) * V + k, vmin, vmax, bad);
        }
    }
    for (; b < nv; b += nt) {
        const uint4 w = __ldcs(xv + b);
        const InT *e = reinterpret_cast<const InT *>(&w);
#pragma unroll
        for (int k = 0; k < V; k++) fr_take<InT>(e[k], b * V + k, vmin, vmax, bad);
    }
    for (uint64_t i = nv * V + tid; i < n; i += nt) fr_take<InT>(x[i], i, vmin, vmax, bad);
    double dmin = (double)vmin, dmax = (double)vmax;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        dmin = fmin(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
        dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
        unsigned long long ob = __shfl_xor_sync(0xffffffffu, bad, o);
        bad = ob < bad ? ob : bad;
    }
    if (lane_id() == 0) {
        if (dmin <= dmax) {
            atomicMin(&mm[0], dkey(dmin));
            atomicMax(&mm[1], dkey(dmax));
        }
        if (bad != ~0ull) atomicMin(&mm[2], bad);
    }
}

// ---- quality statistics (P/pipeline.py:329-345), deterministic sums ----
template <typename InT>
__global__ void k_quality(const InT *a, const InT *b, uint64_t n, double *part_sq,
                          unsigned long long *maxkey) {
    __shared__ double s_w[32];
    double sq = 0.0, mx = 0.0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        double d = (double)a[i] - (double)b[i];
        sq = __dadd_rn(sq, __dmul_rn(d, d));
        mx = fmax(mx, fabs(d));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sq = __dadd_rn(sq, __shfl_xor_sync(0xffffffffu, sq, o));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane_id() == 0) {
        s_w[threadIdx.x >> 5] = sq;
        atomicMax(maxkey, dkey(mx));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (uint32_t w = 0; w < blockDim.x / 32; w++) t = __dadd_rn(t, s_w[w]);
        part_sq[blockIdx.x] = t;
    }
}

__global__ void k_quality_finish(const double *part_sq, uint32_t nparts, const unsigned long long *maxkey,
                                 lzb_dstatus *st) {
    if (threadIdx.x != 0) return;
    double t = 0.0;
    for (uint32_t i = 0; i < nparts; i++) t = __dadd_rn(t, part_sq[i]);
    st->u[0] = __double_as_longlong(dunkey(*maxkey));
    st->u[1] = __double_as_longlong(t);
}

static int nsms() {
    int dev = 0, s = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
    return s > 0 ? s : 148;
}

struct RcLayout {
    bool fast3d;
    bool fast2d;
    bool fast1d;
    bool box;
    uint32_t K;
    uint64_t tiles_per_row, ntiles;
};

static RcLayout rc_layout(const Geom &g) {
    RcLayout L;
    uint64_t vol = g.cx * g.cy * g.cz;
    L.fast3d = g.cx == 8 && g.cy == 8 && g.cz == 8;
    L.fast2d = g.cx == 16 && g.cy == 16 && g.cz == 1 && g.nz == 1;
    L.fast1d = g.cx == 256 && g.cy == 1 && g.cz == 1 && g.ny == 1 && g.nz == 1;
    if (L.fast3d || L.fast2d || L.fast1d) {
        L.box = true;
        L.K = 0;
        L.tiles_per_row = 0;
        L.ntiles = (g.nbx * g.nby * g.nbz + kR3TileChunks - 1) / kR3TileChunks;
        return L;
    }
    L.box = vol >= 1 && vol <= (uint64_t)kRcTile;
    if (L.box) {
        L.K = (uint32_t)(kRcTile / vol);
        L.tiles_per_row = (g.nbx + L.K - 1) / L.K;
        L.ntiles = L.tiles_per_row * g.nby * g.nbz;
    } else {
        L.K = 0;
        L.tiles_per_row = 0;
        L.ntiles = 0;
    }
    return L;
}

template <typename S>
static void rc_scratch(S &s, const Geom &g, const RcLayout &L, uint64_t n_out) {
    s.template take<unsigned long long>(4);
    s.template take<unsigned int>(4);
    if (L.box) {
        s.template take<uint32_t>(L.ntiles + 1);
        s.template take<uint32_t>(L.ntiles + 1);
        s.template take<uint64_t>(L.ntiles + 1);
        s.template take<uint64_t>((L.ntiles + 1 + 2047) / 2048 + 1);
        s.template take<uint64_t>(2 * (n_out ? n_out : 1));
    } else {
        s.template take<int64_t>(g.nx * g.ny * g.nz);
    }
}

}  // namespace lzb

using namespace lzb;

extern "C" size_t lzb_reconstruct_scratch_bytes(const lzb_geom *gg, uint64_t n_out) {
    if (!gg) return 0;
    Geom g = make_geom(*gg);
    ScratchSize s;
    rc_scratch(s, g, rc_layout(g), n_out);
    return s.bytes();
}

extern "C" int lzb_reconstruct(const void *codes, int code_bytes, const uint8_t *outliers,
                               uint64_t n_out, const lzb_geom *gg, double eb_abs, uint32_t cap,
                               void *y, int dtype, int64_t *prequant_out, lzb_dstatus *st,
                               void *scratch, size_t scratch_bytes, void *stream) {
    if (!gg || !codes || !y || !st || (code_bytes != 2 && code_bytes != 4) ||
        (dtype != 0 && dtype != 1) || cap < 4)
        return LZB_E_ARG;
    if (n_out && !outliers) return LZB_E_ARG;
    cudaStream_t s = as_stream(stream);
    Geom g = make_geom(*gg);
    RcLayout L = rc_layout(g);
    Scratch sc(scratch, scratch_bytes);
    unsigned long long *mm = sc.take<unsigned long long>(4);
    unsigned int *tick = sc.take<unsigned int>(4);
    if (!tick) return LZB_E_ARG;
    LZB_CUDA_TRY(cudaMemsetAsync(st, 0, sizeof(lzb_dstatus), s));
    k_mm_init<<<1, 32, 0, s>>>(mm, 4);
    LZB_LAUNCH_CHECK();
    LZB_CUDA_TRY(cudaMemsetAsync(tick, 0, 4 * sizeof(unsigned int), s));
    const int sm = nsms();
    const uint64_t n = g.nx * g.ny * g.nz;
    if (L.box) {
        uint32_t *tile_cnt = sc.take<uint32_t>(L.ntiles + 1);
        uint32_t *tile_fill = sc.take<uint32_t>(L.ntiles + 1);
        uint64_t *tile_start = sc.take<uint64_t>(L.ntiles + 1);
        uint64_t *lb = sc.take<uint64_t>((L.ntiles + 1 + 2047) / 2048 + 1);
        uint64_t *brec = sc.take<uint64_t>(2 * (n_out ? n_out : 1));
        if (!brec) return LZB_E_ARG;
        LZB_CUDA_TRY(cudaMemsetAsync(tile_cnt, 0, (L.ntiles + 1) * sizeof(uint32_t), s));
        LZB_CUDA_TRY(cudaMemsetAsync(tile_fill, 0, (L.ntiles + 1) * sizeof(uint32_t), s));
        LZB_CUDA_TRY(cudaMemsetAsync(lb, 0, ((L.ntiles + 1 + 2047) / 2048 + 1) * sizeof(uint64_t), s));
        OutParams op;
        op.rec = outliers;
        op.n_out = n_out;
        op.fast3d = L.fast3d;
        op.fast2d = L.fast2d;
        op.fast1d = L.fast1d;
        op.tshift = 3;
        op.g = g;
        op.K = L.K;
        op.tiles_per_row = L.tiles_per_row;
        op.ntiles = L.ntiles;
        op.tile_cnt = tile_cnt;
        op.tile_fill = tile_fill;
        op.tile_start = tile_start;
        op.brec = brec;
        op.st = st;
        unsigned go = (unsigned)umin64((n_out + 255) / 256, (uint64_t)sm * 8);
        if (n_out) {
            k_out_count<<<go, 256, 0, s>>>(op);
            LZB_LAUNCH_CHECK();
        }
        k_scan_tiles<<<(unsigned)umin64((L.ntiles + 1 + 2047) / 2048, (uint64_t)sm * 4), 256, 0, s>>>(
            tile_cnt, tile_start, L.ntiles, lb, &tick[0]);
        LZB_LAUNCH_CHECK();
        if (n_out) {
            k_out_scatter<<<go, 256, 0, s>>>(op);
            LZB_LAUNCH_CHECK();
        }
        if (L.fast3d || L.fast2d || L.fast1d) {
            R3Params r3;
            r3.codes = codes;
            r3.g = g;
            r3.two_eb = 2.0 * eb_abs;
            r3.r = (int32_t)(cap / 2);
            r3.y = y;
            r3.pre = prequant_out;
            r3.st = st;
            r3.mm = mm;
            r3.nchunks = g.nbx * g.nby * g.nbz;
            r3.ntiles = L.ntiles;
            r3.tile_start = tile_start;
            r3.brec = brec;
            r3.ticket = &tick[1];
            const size_t osz = dtype == 0 ? 4 : 8;
            r3.vec_ok = (g.nx % (16 / osz) == 0) && ((reinterpret_cast<uintptr_t>(y) & 15) == 0);
            r3.codes_vec = (reinterpret_cast<uintptr_t>(codes) & 15) == 0;
            if (L.fast1d) r3.vec_ok = (reinterpret_cast<uintptr_t>(y) & 15) == 0;  // chunks start at 256 k
            // f32 output through TMA tensor stores (8x8x8 boxes) when the
            // driver exposes the tensor-map encoder and no int64 copy is asked for
            CUtensorMap ymap;
            memset(&ymap, 0, sizeof(ymap));
            bool tma = L.fast3d && dtype == 0 && !prequant_out && r3.vec_ok && tma_encode() != nullptr;
            if (tma) {
                cuuint64_t dims[3] = {g.nx, g.ny, g.nz};
                cuuint64_t strides[2] = {g.nx * 4, g.nx * g.ny * 4};
                cuuint32_t box[3] = {8, 8, 8};
                cuuint32_t estr[3] = {1, 1, 1};
                tma = tma_encode()(&ymap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, y, dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
            }
            const size_t ysm = tma ? (size_t)kR3Warps * 4096 : 0;
            auto launch = [&](auto kern) -> int {
                if (ysm) LZB_CUDA_TRY(set_dyn_smem(kern, ysm));
                int per_sm = 0;
                LZB_CUDA_TRY(occupancy(&per_sm, kern, kR3Threads, ysm));
                if (per_sm < 1) per_sm = 1;
                uint64_t grid = umin64((uint64_t)sm * per_sm, (L.ntiles + kR3Warps - 1) / kR3Warps);
                kern<<<(unsigned)(grid ? grid : 1), kR3Threads, ysm, s>>>(r3, ymap);
                LZB_LAUNCH_CHECK();
                return LZB_OK;
            };
            auto launch2d = [&](auto kern) -> int {
                int per_sm = 0;
                LZB_CUDA_TRY(occupancy(&per_sm, kern, kR3Threads, 0));
                if (per_sm < 1) per_sm = 1;
                uint64_t grid = umin64((uint64_t)sm * per_sm, (L.ntiles + kR3Warps - 1) / kR3Warps);
                kern<<<(unsigned)(grid ? grid : 1), kR3Threads, 0, s>>>(r3);
                LZB_LAUNCH_CHECK();
                return LZB_OK;
            };
            int rc;
            if (L.fast2d)
                rc = code_bytes == 2 ? (dtype == 0 ? launch2d(k_reconstruct_r8<2, uint16_t, float>)
                                                   : launch2d(k_reconstruct_r8<2, uint16_t, double>))
                                     : (dtype == 0 ? launch2d(k_reconstruct_r8<2, uint32_t, float>)
                                                   : launch2d(k_reconstruct_r8<2, uint32_t, double>));
            else if (L.fast1d)
                rc = code_bytes == 2 ? (dtype == 0 ? launch2d(k_reconstruct_r8<1, uint16_t, float>)
                                                   : launch2d(k_reconstruct_r8<1, uint16_t, double>))
                                     : (dtype == 0 ? launch2d(k_reconstruct_r8<1, uint32_t, float>)
                                                   : launch2d(k_reconstruct_r8<1, uint32_t, double>));
            else if (code_bytes == 2)
                rc = dtype == 0 ? (tma ? launch(k_reconstruct3d8<uint16_t, float, true>)
                                       : launch(k_reconstruct3d8<uint16_t, float, false>))
                                : launch(k_reconstruct3d8<uint16_t, double, false>);
            else
                rc = dtype == 0 ? (tma ? launch(k_reconstruct3d8<uint32_t, float, true>)
                                       : launch(k_reconstruct3d8<uint32_t, float, false>))
                                : launch(k_reconstruct3d8<uint32_t, double, false>);
            if (rc) return rc;
            unsigned gf = (unsigned)umin64((n + 255) / 256, (uint64_t)sm * 8);
            if (dtype == 0) k_first_nonfinite<float><<<gf, 256, 0, s>>>((const float *)y, n, mm);
            else k_first_nonfinite<double><<<gf, 256, 0, s>>>((const double *)y, n, mm);
            LZB_LAUNCH_CHECK();
            k_rc_finish<<<1, 1, 0, s>>>(st, mm);
            LZB_LAUNCH_CHECK();
            return LZB_OK;
        }
        RcParams rp;
        rp.codes = codes;
        rp.g = g;
        rp.two_eb = 2.0 * eb_abs;
        rp.radius = cap / 2;
        rp.cap = cap;
        rp.y = y;
        rp.pre = prequant_out;
        rp.st = st;
        rp.mm = mm;
        rp.K = L.K;
        rp.tiles_per_row = L.tiles_per_row;
        rp.ntiles = L.ntiles;
        rp.tile_start = tile_start;
        rp.brec = brec;
        unsigned grid = (unsigned)umin64(L.ntiles, (uint64_t)sm * 8);
        if (code_bytes == 2) {
            if (dtype == 0) k_reconstruct<uint16_t, float><<<grid, kRcThreads, 0, s>>>(rp);
            else k_reconstruct<uint16_t, double><<<grid, kRcThreads, 0, s>>>(rp);
        } else {
            if (dtype == 0) k_reconstruct<uint32_t, float><<<grid, kRcThreads, 0, s>>>(rp);
            else k_reconstruct<uint32_t, double><<<grid, kRcThreads, 0, s>>>(rp);
        }
        LZB_LAUNCH_CHECK();
    } else {
        int64_t *q = sc.take<int64_t>(n);
        if (!q) return LZB_E_ARG;
        unsigned grid = (unsigned)umin64((n + 255) / 256, (uint64_t)sm * 16);
        k_gen_fuse<<<grid, 256, 0, s>>>(codes, code_bytes, g, cap / 2, q);
        LZB_LAUNCH_CHECK();
        if (n_out) {
            k_gen_outliers<<<(unsigned)umin64((n_out + 255) / 256, (uint64_t)sm * 8), 256, 0, s>>>(
                outliers, n_out, n, q, st);
            LZB_LAUNCH_CHECK();
        }
        uint64_t nch = g.nbx * g.nby * g.nbz;
        k_gen_psum<<<(unsigned)umin64((nch + 127) / 128, (uint64_t)sm * 8), 128, 0, s>>>(g, q, st);
        LZB_LAUNCH_CHECK();
        if (dtype == 0)
            k_gen_dequant<float><<<grid, 256, 0, s>>>(q, n, 2.0 * eb_abs, (float *)y, prequant_out, mm);
        else
            k_gen_dequant<double><<<grid, 256, 0, s>>>(q, n, 2.0 * eb_abs, (double *)y, prequant_out, mm);
        LZB_LAUNCH_CHECK();
    }
    k_rc_finish<<<1, 1, 0, s>>>(st, mm);
    LZB_LAUNCH_CHECK();
    return LZB_OK;
}

extern "C" int lzb_dequantize(const int64_t *q, uint64_t n, double eb_abs, void *y, int dtype,
                              lzb_dstatus *st, void *stream) {
    if (!st || (dtype != 0 && dtype != 1)) return LZB_E_ARG;
    cudaStream_t s = as_stream(stream);
    LZB_CUDA_TRY(cudaMemsetAsync(st, 0, sizeof(lzb_dstatus), s));
    unsigned long long *mm = reinterpret_cast<unsigned long long *>(&st->u[3]);
    k_mm_init<<<1, 32, 0, s>>>(mm, 3);
    LZB_LAUNCH_CHECK();
    if (n) {
        if (!q || !y) return LZB_E_ARG;
        unsigned grid = (unsigned)umin64((n + 255) / 256, (uint64_t)nsms() * 8);
        if (dtype == 0) k_gen_dequant<float><<<grid, 256, 0, s>>>(q, n, 2.0 * eb_abs, (float *)y, nullptr, mm);
        else k_gen_dequant<double><<<grid, 256, 0, s>>>(q, n, 2.0 * eb_abs, (double *)y, nullptr, mm);
        LZB_LAUNCH_CHECK();
    }
    k_rc_finish<<<1, 1, 0, s>>>(st, mm);
    LZB_LAUNCH_CHECK();
    return LZB_OK;
}

extern "C" int lzb_field_range(const void *x, int dtype, uint64_t n, lzb_dstatus *st, void *stream) {
    if (!x || !st || (dtype != 0 && dtype != 1)) return LZB_E_ARG;
    cudaStream_t s = as_stream(stream);
    LZB_CUDA_TRY(cudaMemsetAsync(st, 0, sizeof(lzb_dstatus), s));
    // the status block's u[3..5] double as the reduction slots
    unsigned long long *mm = reinterpret_cast<unsigned long long *>(&st->u[3]);
    k_mm_init<<<1, 32, 0, s>>>(mm, 3);
    LZB_LAUNCH_CHECK();
    const int sm = nsms();
    unsigned grid = (unsigned)umin64((n + 255) / 256, (uint64_t)sm * 8);
    if (grid == 0) grid = 1;
    if (dtype == 0) k_field_range<float><<<grid, 256, 0, s>>>((const float *)x, n, mm);
    else k_field_range<double><<<grid, 256, 0, s>>>((const double *)x, n, mm);
    LZB_LAUNCH_CHECK();
    k_rc_finish<<<1, 1, 0, s>>>(st, mm);
    LZB_LAUNCH_CHECK();
    return LZB_OK;
}

extern "C" size_t lzb_quality_scratch_bytes(uint64_t n) {
    (void)n;
    ScratchSize s;
    s.take<double>(4096);
    s.take<unsigned long long>(2);
    return s.bytes();
}

extern "C" int lzb_quality(const void *a, const void *b, int dtype, uint64_t n, lzb_dstatus *st,
                           void *scratch, size_t scratch_bytes, void *stream) {
    if (!a || !b || !st || (dtype != 0 && dtype != 1)) return LZB_E_ARG;
    cudaStream_t s = as_stream(stream);
    Scratch sc(scratch, scratch_bytes);
    double *part = sc.take<double>(4096);
    unsigned long long *mk = sc.take<unsigned long long>(2);
    if (!mk) return LZB_E_ARG;
    LZB_CUDA_TRY(cudaMemsetAsync(st, 0, sizeof(lzb_dstatus), s));
    LZB_CUDA_TRY(cudaMemsetAsync(mk, 0, 2 * sizeof(unsigned long long), s));
    unsigned grid = (unsigned)umin64((n + 255) / 256, 4096);
    if (grid == 0) grid = 1;
    if (dtype == 0) k_quality<float><<<grid, 256, 0, s>>>((const float *)a, (const float *)b, n, part, mk);
    else k_quality<double><<<grid, 256, 0, s>>>((const double *)a, (const double *)b, n, part, mk);
    LZB_LAUNCH_CHECK();
    k_quality_finish<<<1, 32, 0, s>>>(part, grid, mk, st);
    LZB_LAUNCH_CHECK();
    return LZB_OK;
}

extern "C" const char *lzb_version(void) { return "lzb 0.1.0 sm_100a"; }

extern "C" const char *lzb_strerror(int code) {
    switch (code) {
        case LZB_OK: return "ok";
        case LZB_E_ARG: return "invalid argument";
        case LZB_E_DATA: return "data error";
        case LZB_E_OVERFLOW: return "quantization overflow";
        case LZB_E_CORRUPT: return "corrupt archive";
        case LZB_E_CUDA: return "CUDA error";
        case LZB_E_ASSERT: return "error-bound invariant violated";
        case LZB_E_CAPACITY: return "output capacity exceeded";
        default: return "unknown";
    }
}

// ---------------------------------------------------------------------------
// Byte copy by SMs (not a copy engine): with unified addressing a pinned host
// buffer is readable / writable from kernels, so a host<->device copy done
// this way runs beside the DMA queues instead of behind them.
namespace lzb {
__global__ void __launch_bounds__(256) k_copy_bytes(uint8_t *dst, const uint8_t *src, uint64_t n) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const bool vec = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0;
    uint64_t done = 0;
    if (vec) {
        const uint64_t nv = n / 16;
        const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
        uint4 *d4 = reinterpret_cast<uint4 *>(dst);
        for (uint64_t i = i0; i < nv; i += stride) d4[i] = s4[i];
        done = nv * 16;
    }
    for (uint64_t i = done + i0; i < n; i += stride) dst[i] = src[i];
}
}  // namespace lzb


extern "C" int lzb_copy_bytes(void *dst, const void *src, uint64_t n, void *stream) {
    if (n == 0) return LZB_OK;
    if (!dst || !src) return LZB_E_ARG;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t blocks = umin64((n / 16 + 255) / 256 + 1, (uint64_t)sms * 4);
    lzb::k_copy_bytes<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(static_cast<uint8_t *>(dst),
                                                                     static_cast<const uint8_t *>(src), n);
    LZB_LAUNCH_CHECK();
    return LZB_OK;
}
