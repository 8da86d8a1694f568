// K1: fused prequantization + chunk-local Lorenzo delta + quant code +
// histogram + outlier gather, writing the chunk-major symbol stream.
//
// Reference semantics (P = /root/reference/pkg/src/lzebc):
//   prequantize            P/quantize.py:90-110
//   _lorenzo_deltas        P/quantize.py:136-141  (nested first differences,
//                           zero prepend INSIDE each chunk -- no halo)
//   construct_chunk        P/quantize.py:144-158
//   construct_grid         P/quantize.py:161-193  (outliers sorted by global index)
//   gather_chunk_major     P/pipeline.py:102-105
//   histogram              P/codebook.py:23-27
//
// Design (K1): persistent CTAs claim tiles by ticket.  A tile is up
// to K whole chunks adjacent along x inside one chunk row, so it is one
// contiguous box of the input AND one contiguous range of the chunk-major
// stream.  The box is read once, coalesced, prequantized in f64 into shared
// memory; deltas are formed from shared memory; codes are staged and written
// back as one contiguous vectorised range.  The histogram is privatised per
// CTA in shared memory for the whole persistent loop.  Outliers are compacted
// in stream order (block scan + decoupled look-back over tiles), i.e. in
// chunk-major order; a device-side check + stable per-chunk-row reorder turns
// that into the archive's global row-major order only when needed.
#include <type_traits>

#include "lzb_common.cuh"
#include "lzb_quant3d.cuh"
#include "lzb_quant3t.cuh"
#include "lzb_quant2d.cuh"

namespace lzb {

constexpr int kQThreads = 256;
constexpr int kTile = 4096;  // max elements per tile (16 per thread)
constexpr int kSeg = kTile / kQThreads;
constexpr uint32_t kSmemHistMaxCap = 4096;
constexpr double kPrequantLimit = 576460752303423488.0;  // 2^59, P/quantize.py:22

struct QuantParams {
    const void *x;
    Geom g;
    double two_eb;
    double slack;  // eb_abs * (1 + 1e-12)  (P/quantize.py:108-111)
    float inv_hi, inv_lo;  // 1 / two_eb as a float pair (f32 fast prequant)
    int64_t radius;
    uint32_t cap;
    void *codes;
    unsigned long long *hist;
    uint64_t *records;  // {u64 index, i64 delta} pairs, chunk-major order
    uint64_t out_capacity;
    lzb_dstatus *st;
    uint64_t *lb;        // look-back status per tile
    unsigned int *ticket;
    uint64_t ntiles;
    // box mode
    uint32_t K;              // chunks per tile
    uint64_t tiles_per_row;  // ceil(nbx / K)
};

// f64 prequantization, bit-identical with numpy (P/quantize.py:90-110).
// Returns false on overflow; sets *bad when the debug-assert invariant fails.
__device__ __forceinline__ int64_t prequant(double v, double two_eb, double slack, int &flags) {
    double s = __ddiv_rn(v, two_eb);
    double r = trunc(__dadd_rn(s, copysign(0.5, s)));
    if (fabs(r) >= kPrequantLimit) {
        flags |= 1;
        return 0;
    }
    int64_t c = (int64_t)r;
    double back = __dmul_rn((double)c, two_eb);
    if (!(fabs(__dsub_rn(v, back)) <= slack)) flags |= 2;
    return c;
}

template <typename InT>
__device__ __forceinline__ double load_in(const void *x, uint64_t i) {
    return (double)static_cast<const InT *>(x)[i];
}

// value at element i as a prequant integer: float inputs are prequantized,
// int64 inputs (dtype 2, construct_grid on a PrequantGrid) are taken as is.
template <typename InT>
__device__ __forceinline__ int64_t load_pre(const QuantParams &p, uint64_t i, int &flags) {
    if constexpr (std::is_same<InT, int64_t>::value) {
        return static_cast<const int64_t *>(p.x)[i];
    } else if constexpr (std::is_same<InT, float>::value) {
        // f32: the double-single fast path of K1's 3D kernels (same proof,
        // DESIGN.md K1); exact f64 division only near a rounding tie / 2^22
        const float xv = static_cast<const float *>(p.x)[i];
        bool ok = true;
        const int32_t d = f3::pq_fast_f32(xv, p.inv_hi, p.inv_lo, ok);
        if (ok) return d;
        return prequant((double)xv, p.two_eb, p.slack, flags);
    } else {
        return prequant(load_in<InT>(p.x, i), p.two_eb, p.slack, flags);
    }
}

// Tile geometry in box mode.
struct BoxTile {
    uint64_t X0, Y0, Z0;
    uint32_t BX, EY, EZ;   // box extents
    uint32_t kc;           // chunks in this tile
    uint32_t cx;           // chunk edge x
    uint32_t last_ex;      // x extent of the last chunk of the tile
    uint64_t stream_base;  // chunk-major offset of the tile's first element
    uint32_t n;            // elements
};

__device__ __forceinline__ BoxTile box_tile(const QuantParams &p, uint64_t t) {
    const Geom &g = p.g;
    uint64_t row = t / p.tiles_per_row, j = t - row * p.tiles_per_row;
    uint64_t bx0 = j * p.K, by = row % g.nby, bz = row / g.nby;
    BoxTile b;
    b.kc = (uint32_t)umin64(p.K, g.nbx - bx0);
    b.X0 = bx0 * g.cx;
    b.Y0 = by * g.cy;
    b.Z0 = bz * g.cz;
    b.BX = (uint32_t)umin64(b.kc * g.cx, g.nx - b.X0);
    b.EY = (uint32_t)umin64(g.cy, g.ny - b.Y0);
    b.EZ = (uint32_t)umin64(g.cz, g.nz - b.Z0);
    b.cx = (uint32_t)g.cx;
    b.last_ex = b.BX - (b.kc - 1) * b.cx;
    b.stream_base = chunk_base(g, bx0, by, bz);
    b.n = b.BX * b.EY * b.EZ;
    return b;
}

// stream position inside a box tile -> box coordinates + chunk-local coords
__device__ __forceinline__ void box_pos(const BoxTile &b, uint32_t p, uint32_t &bxl, uint32_t &ly,
                                        uint32_t &lz, uint32_t &lx) {
    uint32_t full = b.cx * b.EY * b.EZ;
    uint32_t k = p / full;
    uint32_t r = p - k * full;
    uint32_t ex = (k == b.kc - 1) ? b.last_ex : b.cx;
    uint32_t exy = ex * b.EY;
    lz = r / exy;
    r -= lz * exy;
    ly = r / ex;
    lx = r - ly * ex;
    bxl = k * b.cx + lx;
}

// chunk-local Lorenzo delta from the prequant box (zero outside the chunk).
__device__ __forceinline__ int64_t box_delta(const int64_t *s, const BoxTile &b, uint32_t bxl,
                                             uint32_t ly, uint32_t lz, uint32_t lx) {
    const uint32_t sy = b.BX, sz = b.BX * b.EY;
    const uint32_t i = bxl + sy * ly + sz * lz;
    int64_t d = s[i];
    const bool hx = lx > 0, hy = ly > 0, hz = lz > 0;
    if (hx) d -= s[i - 1];
    if (hy) d -= s[i - sy];
    if (hx && hy) d += s[i - 1 - sy];
    if (hz) {
        d -= s[i - sz];
        if (hx) d += s[i - 1 - sz];
        if (hy) d += s[i - sy - sz];
        if (hx && hy) d -= s[i - 1 - sy - sz];
    }
    return d;
}

// Generic stream position -> coordinates (any ChunkSpec).
struct StreamCoord {
    uint64_t x, y, z;
    uint64_t lx, ly, lz;
};

__device__ __forceinline__ StreamCoord stream_coord(const Geom &g, uint64_t pos) {
    StreamCoord c;
    uint64_t layer = g.nx * g.ny * g.cz;
    uint64_t bz = pos / layer;
    uint64_t r = pos - bz * layer;
    uint64_t ez = umin64(g.cz, g.nz - bz * g.cz);
    uint64_t rowsz = g.nx * ez * g.cy;
    uint64_t by = r / rowsz;
    r -= by * rowsz;
    uint64_t ey = umin64(g.cy, g.ny - by * g.cy);
    uint64_t csz = ez * ey * g.cx;
    uint64_t bx = r / csz;
    r -= bx * csz;
    uint64_t ex = umin64(g.cx, g.nx - bx * g.cx);
    c.lz = r / (ex * ey);
    r -= c.lz * ex * ey;
    c.ly = r / ex;
    c.lx = r - c.ly * ex;
    c.x = bx * g.cx + c.lx;
    c.y = by * g.cy + c.ly;
    c.z = bz * g.cz + c.lz;
    return c;
}

template <typename InT>
__device__ __forceinline__ int64_t stream_delta(const QuantParams &p, const StreamCoord &c,
                                                int &flags) {
    const Geom &g = p.g;
    const uint64_t i = c.x + g.nx * (c.y + g.ny * c.z);
    const uint64_t sy = g.nx, sz = g.nx * g.ny;
    auto pq = [&](uint64_t j) { return load_pre<InT>(p, j, flags); };
    int64_t d = pq(i);
    const bool hx = c.lx > 0, hy = c.ly > 0, hz = c.lz > 0;
    if (hx) d -= pq(i - 1);
    if (hy) d -= pq(i - sy);
    if (hx && hy) d += pq(i - 1 - sy);
    if (hz) {
        d -= pq(i - sz);
        if (hx) d += pq(i - 1 - sz);
        if (hy) d += pq(i - sy - sz);
        if (hx && hy) d -= pq(i - 1 - sy - sz);
    }
    return d;
}

template <typename InT, typename SymT, bool BOX>
__global__ void __launch_bounds__(kQThreads) k_quantize(QuantParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // layout: [s_pre int64 kTile (BOX only)] [s_code SymT kTile] [s_bits u32 kTile/32] [s_hist u32 cap]
    int64_t *s_pre = reinterpret_cast<int64_t *>(smem_raw);
    SymT *s_code = reinterpret_cast<SymT *>(smem_raw + (BOX ? kTile * sizeof(int64_t) : 0));
    uint32_t *s_bits = reinterpret_cast<uint32_t *>(reinterpret_cast<unsigned char *>(s_code) +
                                                    kTile * sizeof(SymT));
    uint32_t *s_hist = s_bits + kTile / 32;
    __shared__ uint64_t s_tile, s_excl;
    __shared__ uint32_t s_scan[33];

    const bool smem_hist = p.cap <= kSmemHistMaxCap;
    if (smem_hist)
        for (uint32_t i = threadIdx.x; i < p.cap; i += blockDim.x) s_hist[i] = 0;
    const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
    const int64_t r = p.radius;
    int flags = 0;
    const bool line = p.g.ny == 1 && p.g.nz == 1;  // 1D geometry: no index divisions
    const bool cx_pow2 = (p.g.cx & (p.g.cx - 1)) == 0;

    while (true) {
        if (tid == 0) s_tile = atomicAdd(p.ticket, 1u);
        __syncthreads();
        const uint64_t t = s_tile;
        if (t >= p.ntiles) break;

        BoxTile b;
        uint64_t base;
        uint32_t n;
        if (BOX) {
            b = box_tile(p, t);
            base = b.stream_base;
            n = b.n;
            // ---- load + prequantize the box (coalesced along x) ----
            const uint32_t bxy = b.BX * b.EY;
            if (line) {  // 1D: the box is a contiguous range of the field
                for (uint32_t i = tid; i < n; i += kQThreads) s_pre[i] = load_pre<InT>(p, b.X0 + i, flags);
            } else {
                for (uint32_t i = tid; i < n; i += kQThreads) {
                    uint32_t z = i / bxy, rem = i - z * bxy, y = rem / b.BX, xx = rem - y * b.BX;
                    uint64_t gi = (b.X0 + xx) + p.g.nx * ((b.Y0 + y) + p.g.ny * (b.Z0 + z));
                    s_pre[i] = load_pre<InT>(p, gi, flags);
                }
            }
            __syncthreads();
        } else {
            base = t * (uint64_t)kTile;
            uint64_t total = p.g.nx * p.g.ny * p.g.nz;
            n = (uint32_t)umin64(kTile, total - base);
        }

        // ---- deltas -> codes (staged), outlier bitmap, histogram ----
        for (uint32_t j = 0; j < (uint32_t)kTile; j += kQThreads) {
            const uint32_t pos = j + tid;
            bool outl = false;
            if (pos < n) {
                int64_t d;
                if (BOX && line) {  // 1D: first difference inside the chunk
                    const uint32_t lx = cx_pow2 ? (pos & (b.cx - 1)) : pos % b.cx;
                    d = s_pre[pos] - (lx ? s_pre[pos - 1] : 0);
                } else if (BOX) {
                    uint32_t bxl, ly, lz, lx;
                    box_pos(b, pos, bxl, ly, lz, lx);
                    d = box_delta(s_pre, b, bxl, ly, lz, lx);
                } else {
                    d = stream_delta<InT>(p, stream_coord(p.g, base + pos), flags);
                }
                int64_t ad = d < 0 ? -d : d;
                uint32_t code;
                if (ad < r) {
                    code = (uint32_t)(d + r);
                } else {
                    code = (uint32_t)r;
                    outl = true;
                }
                s_code[pos] = (SymT)code;
                if (smem_hist)
                    atomicAdd(&s_hist[code], 1u);
                else
                    atomicAdd(&p.hist[code], 1ull);
            }
            uint32_t bal = __ballot_sync(0xffffffffu, outl);
            if (lane == 0) s_bits[(j >> 5) + warp] = bal;
        }
        __syncthreads();

        // ---- write the codes: one contiguous stream range ----
        SymT *out = static_cast<SymT *>(p.codes) + base;
        constexpr uint32_t kVec = 16 / sizeof(SymT);
        if ((reinterpret_cast<uintptr_t>(out) & 15) == 0 && (n % kVec) == 0) {
            const uint4 *src = reinterpret_cast<const uint4 *>(s_code);
            uint4 *dst = reinterpret_cast<uint4 *>(out);
            for (uint32_t i = tid; i < n / kVec; i += kQThreads) dst[i] = src[i];
        } else {
            for (uint32_t i = tid; i < n; i += kQThreads) out[i] = s_code[i];
        }

        // ---- outliers in stream order: thread owns positions [tid*kSeg, +kSeg) ----
        const uint32_t seg0 = tid * kSeg;
        uint32_t segbits = (s_bits[seg0 >> 5] >> (seg0 & 31)) & ((1u << kSeg) - 1u);
        uint32_t cnt = __popc(segbits);
        uint32_t total;
        uint32_t off = block_exclusive_scan<uint32_t>(cnt, s_scan, &total);
        if (warp == 0) {
            uint64_t ex = lookback_warp(p.lb, t, total);
            if (lane == 0) s_excl = ex;
        }
        __syncthreads();
        const uint64_t excl = s_excl;
        uint64_t w = excl + off;
        while (segbits) {
            uint32_t bit = __ffs(segbits) - 1;
            segbits &= segbits - 1;
            uint32_t pos = seg0 + bit;
            int64_t d;
            uint64_t gi;
            if (BOX) {
                uint32_t bxl, ly, lz, lx;
                box_pos(b, pos, bxl, ly, lz, lx);
                d = box_delta(s_pre, b, bxl, ly, lz, lx);
                gi = (b.X0 + bxl) + p.g.nx * ((b.Y0 + ly) + p.g.ny * (b.Z0 + lz));
            } else {
                StreamCoord c = stream_coord(p.g, base + pos);
                int dummy = 0;
                d = stream_delta<InT>(p, c, dummy);
                gi = c.x + p.g.nx * (c.y + p.g.ny * c.z);
            }
            if (w < p.out_capacity) {
                p.records[2 * w] = gi;
                p.records[2 * w + 1] = (uint64_t)d;
            }
            w++;
        }
        if (t == p.ntiles - 1 && tid == 0) {
            uint64_t nout = excl + total;
            p.st->u[0] = nout;
            if (nout > p.out_capacity) set_status(p.st, LZB_E_CAPACITY);
        }
        __syncthreads();
    }

    if (smem_hist) {
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < p.cap; i += blockDim.x)
            if (s_hist[i]) atomicAdd(&p.hist[i], (unsigned long long)s_hist[i]);
    }
    flags = __reduce_or_sync(0xffffffffu, flags);
    if (lane == 0 && flags) {
        if (flags & 1) set_status(p.st, LZB_E_OVERFLOW);
        else set_status(p.st, LZB_E_ASSERT);
    }
}

// ----------------------------------------------------------------------------
// Outlier ordering.  Records come out of K1 in chunk-major order.  The
// archive wants them sorted by global row-major index (P/quantize.py:184-193).
// Inside one chunk row (fixed by, bz) the records of one grid row (y, z) are
// already in x order, so a STABLE counting sort by grid row restricted to each
// chunk-row segment -- placed at the global row offsets -- yields the global
// order.  All of this is skipped (device flag) when the records are already
// strictly increasing, which is the common case (smooth fields put outliers
// at chunk origins).
// ----------------------------------------------------------------------------
struct OrderParams {
    uint64_t *records;  // in/out
    uint64_t *tmp;      // copy of records
    const lzb_dstatus *st;
    uint64_t capacity;
    Geom g;
    uint32_t *unsorted;      // flag
    uint32_t *row_cnt;       // ny*nz
    uint64_t *row_start;     // ny*nz
    uint64_t *seg_start;     // per chunk row
    uint64_t *seg_end;       // per chunk row (0 = empty)
    uint64_t *scan_lb;
    unsigned int *scan_ticket;
};

__device__ __forceinline__ uint64_t order_count(const OrderParams &p) {
    uint64_t n = p.st->u[0];
    return n > p.capacity ? 0 : n;  // capacity errors are reported by K1
}

__global__ void k_check_sorted(OrderParams p) {
    const uint64_t n = order_count(p);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i + 1 < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (!(p.records[2 * i] < p.records[2 * (i + 1)])) *p.unsorted = 1u;
    }
}

__device__ __forceinline__ uint64_t chunk_row_of(const Geom &g, uint64_t idx) {
    uint64_t x = idx % g.nx, yz = idx / g.nx;
    (void)x;
    uint64_t y = yz % g.ny, z = yz / g.ny;
    return (y / g.cy) + g.nby * (z / g.cz);
}

__global__ void k_order_prepare(OrderParams p) {
    if (!*p.unsorted) return;
    const uint64_t n = order_count(p);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t idx = p.records[2 * i];
        p.tmp[2 * i] = idx;
        p.tmp[2 * i + 1] = p.records[2 * i + 1];
        atomicAdd(&p.row_cnt[idx / p.g.nx], 1u);
        uint64_t cr = chunk_row_of(p.g, idx);
        if (i == 0 || chunk_row_of(p.g, p.records[2 * (i - 1)]) != cr) p.seg_start[cr] = i;
        if (i + 1 == n || chunk_row_of(p.g, p.records[2 * (i + 1)]) != cr) p.seg_end[cr] = i + 1;
    }
}

// exclusive scan u32 -> u64 with decoupled look-back (1 element per thread x 8)
constexpr int kScanItems = 8;
__global__ void __launch_bounds__(256) k_scan_u32(const uint32_t *in, uint64_t *out, uint64_t n,
                                                  uint64_t *lb, unsigned int *ticket,
                                                  const uint32_t *enable) {
    if (enable && !*enable) return;
    __shared__ uint64_t s_t, s_ex;
    __shared__ uint64_t s_scan[33];
    if (threadIdx.x == 0) s_t = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint64_t t = s_t;
    const uint64_t base = t * 256 * kScanItems + (uint64_t)threadIdx.x * kScanItems;
    uint64_t v[kScanItems];
    uint64_t sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        v[k] = base + k < n ? in[base + k] : 0;
        sum += v[k];
    }
    uint64_t total;
    uint64_t off = block_exclusive_scan<uint64_t>(sum, s_scan, &total);
    if ((threadIdx.x >> 5) == 0) {
        uint64_t ex = lookback_warp(lb, t, total);
        if (lane_id() == 0) s_ex = ex;
    }
    __syncthreads();
    uint64_t run = s_ex + off;
#pragma unroll
    for (int k = 0; k < kScanItems; k++) {
        if (base + k < n) out[base + k] = run;
        run += v[k];
    }
}

// One CTA per chunk row: stable multi-split of its segment by local grid row.
constexpr uint32_t kOrderMaxRows = 1024;
__global__ void __launch_bounds__(256) k_order_scatter(OrderParams p) {
    if (!*p.unsorted) return;
    __shared__ uint32_t s_run[kOrderMaxRows];
    __shared__ uint32_t s_w[8][kOrderMaxRows];
    const Geom &g = p.g;
    const uint64_t nrows_c = g.nby * g.nbz;
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    for (uint64_t cr = blockIdx.x; cr < nrows_c; cr += gridDim.x) {
        const uint64_t s0 = p.seg_start[cr], s1 = p.seg_end[cr];
        if (s1 == 0) continue;
        const uint64_t by = cr % g.nby, bz = cr / g.nby;
        const uint64_t Y0 = by * g.cy, Z0 = bz * g.cz;
        const uint32_t EY = (uint32_t)umin64(g.cy, g.ny - Y0);
        const uint32_t EZ = (uint32_t)umin64(g.cz, g.nz - Z0);
        const uint32_t R = EY * EZ;
        if (R <= kOrderMaxRows) {
            for (uint32_t i = threadIdx.x; i < R; i += blockDim.x) s_run[i] = 0;
            for (uint32_t i = threadIdx.x; i < 8 * R; i += blockDim.x) (&s_w[0][0])[i / R * kOrderMaxRows + i % R] = 0;
            __syncthreads();
            for (uint64_t b0 = s0; b0 < s1; b0 += blockDim.x) {
                const uint64_t i = b0 + threadIdx.x;
                const bool act = i < s1;
                uint32_t lr = 0xffffffffu;
                uint64_t idx = 0;
                if (act) {
                    idx = p.tmp[2 * i];
                    uint64_t yz = idx / g.nx;
                    uint64_t y = yz % g.ny, z = yz / g.ny;
                    lr = (uint32_t)((y - Y0) + EY * (z - Z0));
                }
                uint32_t peers = __match_any_sync(0xffffffffu, lr);
                uint32_t rank = __popc(peers & ((1u << lane) - 1u));
                uint32_t leader = __ffs(peers) - 1;
                if (act && lane == leader) s_w[warp][lr] = __popc(peers);
                __syncthreads();
                if (act) {
                    uint32_t before = s_run[lr];
                    for (uint32_t w2 = 0; w2 < warp; w2++) before += s_w[w2][lr];
                    uint64_t dst = p.row_start[idx / g.nx] + before + rank;
                    // row_start is the global exclusive offset of the grid row;
                    // `before + rank` counts this row's earlier records.
                    p.records[2 * dst] = idx;
                    p.records[2 * dst + 1] = p.tmp[2 * i + 1];
                }
                __syncthreads();
                if (act && lane == leader) {
                    uint32_t c = s_w[warp][lr];
                    atomicAdd(&s_run[lr], c);
                    s_w[warp][lr] = 0;
                }
                __syncthreads();
            }
        } else {
            // very tall chunk rows: thread per grid row, ordered walk of the segment
            for (uint32_t lr = threadIdx.x; lr < R; lr += blockDim.x) {
                uint64_t y = Y0 + lr % EY, z = Z0 + lr / EY;
                uint64_t row = y + g.ny * z;
                uint64_t dst = p.row_start[row];
                for (uint64_t i = s0; i < s1; i++) {
                    uint64_t idx = p.tmp[2 * i];
                    if (idx / g.nx == row) {
                        p.records[2 * dst] = idx;
                        p.records[2 * dst + 1] = p.tmp[2 * i + 1];
                        dst++;
                    }
                }
            }
        }
        __syncthreads();
    }
}

// ----------------------------------------------------------------------------
// host side
// ----------------------------------------------------------------------------
static bool box_mode_ok(const Geom &g, uint32_t *K) {
    uint64_t vol = g.cx * g.cy * g.cz;
    if (vol == 0 || vol > (uint64_t)kTile) return false;
    *K = (uint32_t)(kTile / vol);
    return true;
}

struct QuantLayout {
    uint64_t ntiles;
    bool fast3d;
    bool fast2d;  // ChunkSpec(16,16) on a 2D grid: k_quantize_r8<2>
    bool fast1d;  // ChunkSpec(256) on a 1D grid: k_quantize_r8<1>
    bool box;
    uint32_t K;
    uint64_t tiles_per_row;
    uint64_t nrows_grid, nrows_chunk;
};

static QuantLayout quant_layout(const Geom &g) {
    QuantLayout L;
    uint64_t n = g.nx * g.ny * g.nz;
    L.box = box_mode_ok(g, &L.K);
    if (L.box) {
        L.tiles_per_row = (g.nbx + L.K - 1) / L.K;
        L.ntiles = L.tiles_per_row * g.nby * g.nbz;
    } else {
        L.K = 0;
        L.tiles_per_row = 0;
        L.ntiles = (n + kTile - 1) / kTile;
    }
    L.nrows_grid = g.ny * g.nz;
    L.nrows_chunk = g.nby * g.nbz;
    L.fast3d = g.cx == 8 && g.cy == 8 && g.cz == 8;
    L.fast2d = g.cx == 16 && g.cy == 16 && g.cz == 1 && g.nz == 1;
    L.fast1d = g.cx == 256 && g.cy == 1 && g.cz == 1 && g.ny == 1 && g.nz == 1;
    if (L.fast3d || L.fast2d || L.fast1d) {
        uint64_t nch = g.nbx * g.nby * g.nbz;
        uint64_t nt = (nch + kQ3TileChunks - 1) / kQ3TileChunks;
        if (nt > L.ntiles) L.ntiles = nt;
    }
    return L;
}

template <typename S>
static void quant_scratch(S &s, const QuantLayout &L, uint64_t cap_out) {
    s.template take<uint64_t>(L.ntiles);                 // look-back
    s.template take<unsigned int>(4);                    // tickets + flag
    s.template take<uint64_t>(2 * cap_out);              // reorder copy
    s.template take<uint32_t>(L.nrows_grid);             // row counts
    s.template take<uint64_t>(L.nrows_grid);             // row starts
    s.template take<uint64_t>(L.nrows_chunk);            // seg start
    s.template take<uint64_t>(L.nrows_chunk);            // seg end
    s.template take<uint64_t>((L.nrows_grid + 2047) / 2048 + 1);  // scan look-back
    if (L.fast3d || L.fast2d || L.fast1d) {
        s.template take<uint64_t>(L.ntiles * 2 * kQ3Slot);  // record slots
        s.template take<uint32_t>(L.ntiles);                // tile counts
        s.template take<uint32_t>(L.ntiles);                // overflow list
        s.template take<uint64_t>(L.ntiles);                // tile offsets
        s.template take<uint64_t>((L.ntiles + 2047) / 2048 + 1);  // scan look-back
    }
}

static int device_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = kNumSMs;
    }
    return sms;
}

template <typename InT, typename SymT, bool BOX>
static int launch_quant(const QuantParams &qp, cudaStream_t s) {
    size_t smem = (BOX ? kTile * sizeof(int64_t) : 0) + kTile * sizeof(SymT) + kTile / 8 +
                  (qp.cap <= kSmemHistMaxCap ? qp.cap * sizeof(uint32_t) : 0);
    auto kern = k_quantize<InT, SymT, BOX>;
    LZB_CUDA_TRY(set_dyn_smem(kern, smem));
    int per_sm = 0;
    LZB_CUDA_TRY(occupancy(&per_sm, kern, kQThreads, smem));
    if (per_sm < 1) per_sm = 1;
    uint64_t grid = (uint64_t)device_sms() * per_sm;
    if (grid > qp.ntiles) grid = qp.ntiles ? qp.ntiles : 1;
    kern<<<(unsigned)grid, kQThreads, smem, s>>>(qp);
    LZB_LAUNCH_CHECK();
    return LZB_OK;
}

}  // namespace lzb

using namespace lzb;

extern "C" size_t lzb_quantize_scratch_bytes(const lzb_geom *g, uint64_t out_capacity) {
    if (!g) return 0;
    ScratchSize s;
    quant_scratch(s, quant_layout(make_geom(*g)), out_capacity);
    return s.bytes();
}

static int quantize_impl(const void *x, int dtype, const lzb_geom *gg, double eb_abs, uint32_t cap, void *codes,
                         int code_bytes, uint64_t *hist, uint64_t *outliers, uint64_t out_capacity,
                         lzb_dstatus *st, void *scratch, size_t scratch_bytes, void *stream,
                         cudaEvent_t hist_ev);

extern "C" int lzb_quantize(const void *x, int dtype, const lzb_geom *gg, double eb_abs,
                            uint32_t cap, void *codes, int code_bytes, uint64_t *hist,
                            uint64_t *outliers, uint64_t out_capacity, lzb_dstatus *st,
                            void *scratch, size_t scratch_bytes, void *stream) {
    return quantize_impl(x, dtype, gg, eb_abs, cap, codes, code_bytes, hist, outliers, out_capacity, st, scratch,
                         scratch_bytes, stream, nullptr);
}

extern "C" int lzb_quantize_ev(const void *x, int dtype, const lzb_geom *gg, double eb_abs, uint32_t cap,
                               void *codes, int code_bytes, uint64_t *hist, uint64_t *outliers,
                               uint64_t out_capacity, lzb_dstatus *st, void *scratch, size_t scratch_bytes,
                               void *stream, void *hist_event) {
    return quantize_impl(x, dtype, gg, eb_abs, cap, codes, code_bytes, hist, outliers, out_capacity, st, scratch,
                         scratch_bytes, stream, static_cast<cudaEvent_t>(hist_event));
}

static int quantize_impl(const void *x, int dtype, const lzb_geom *gg, double eb_abs, uint32_t cap, void *codes,
                         int code_bytes, uint64_t *hist, uint64_t *outliers, uint64_t out_capacity,
                         lzb_dstatus *st, void *scratch, size_t scratch_bytes, void *stream,
                         cudaEvent_t hist_ev) {
    if (!gg || !x || !codes || !hist || !st || dtype < 0 || dtype > 2) return LZB_E_ARG;
    if (code_bytes != 2 && code_bytes != 4) return LZB_E_ARG;
    if (cap < 4 || (cap & (cap - 1)) || (code_bytes == 2 && cap > 65536)) return LZB_E_ARG;
    if (gg->cx < 1 || gg->cy < 1 || gg->cz < 1 || gg->nx < 1 || gg->ny < 1 || gg->nz < 1)
        return LZB_E_ARG;
    cudaStream_t s = as_stream(stream);
    Geom g = make_geom(*gg);
    QuantLayout L = quant_layout(g);
    Scratch sc(scratch, scratch_bytes);
    uint64_t *lb = sc.take<uint64_t>(L.ntiles);
    unsigned int *tick = sc.take<unsigned int>(4);
    uint64_t *tmp = sc.take<uint64_t>(2 * out_capacity);
    uint32_t *row_cnt = sc.take<uint32_t>(L.nrows_grid);
    uint64_t *row_start = sc.take<uint64_t>(L.nrows_grid);
    uint64_t *seg_start = sc.take<uint64_t>(L.nrows_chunk);
    uint64_t *seg_end = sc.take<uint64_t>(L.nrows_chunk);
    uint64_t *scan_lb = sc.take<uint64_t>((L.nrows_grid + 2047) / 2048 + 1);
    if (!scan_lb) return LZB_E_ARG;
    uint64_t *slots = nullptr, *tile_off = nullptr, *slb = nullptr;
    uint32_t *tile_cnt = nullptr, *over_list = nullptr;
    if (L.fast3d || L.fast2d || L.fast1d) {
        slots = sc.take<uint64_t>(L.ntiles * 2 * kQ3Slot);
        tile_cnt = sc.take<uint32_t>(L.ntiles);
        over_list = sc.take<uint32_t>(L.ntiles);
        tile_off = sc.take<uint64_t>(L.ntiles);
        slb = sc.take<uint64_t>((L.ntiles + 2047) / 2048 + 1);
        if (!slb) return LZB_E_ARG;
        LZB_CUDA_TRY(cudaMemsetAsync(slb, 0, ((L.ntiles + 2047) / 2048 + 1) * sizeof(uint64_t), s));
    }

    LZB_CUDA_TRY(cudaMemsetAsync(st, 0, sizeof(lzb_dstatus), s));
    LZB_CUDA_TRY(cudaMemsetAsync(hist, 0, cap * sizeof(uint64_t), s));
    LZB_CUDA_TRY(cudaMemsetAsync(lb, 0, L.ntiles * sizeof(uint64_t), s));
    LZB_CUDA_TRY(cudaMemsetAsync(tick, 0, 4 * sizeof(unsigned int), s));

    QuantParams qp;
    qp.x = x;
    qp.g = g;
    qp.two_eb = 2.0 * eb_abs;
    qp.slack = eb_abs * (1.0 + 1e-12);
    {
        const double inv = 1.0 / (2.0 * eb_abs);
        qp.inv_hi = (float)inv;
        qp.inv_lo = (float)(inv - (double)qp.inv_hi);
    }
    qp.radius = cap / 2;
    qp.cap = cap;
    qp.codes = codes;
    qp.hist = reinterpret_cast<unsigned long long *>(hist);
    qp.records = outliers;
    qp.out_capacity = outliers ? out_capacity : 0;
    qp.st = st;
    qp.lb = lb;
    qp.ticket = &tick[0];
    qp.ntiles = L.ntiles;
    qp.K = L.K;
    qp.tiles_per_row = L.tiles_per_row;

    int rc;
    // the register paths store codes with 16-byte vector stores
    const bool codes_vec = (reinterpret_cast<uintptr_t>(codes) & 15) == 0;
    if ((L.fast3d || L.fast2d || L.fast1d) && dtype != 2 && codes_vec) {
        Q3Params q3;
        q3.x = x;
        q3.g = g;
        q3.two_eb = 2.0 * eb_abs;
        q3.inv = 1.0 / (2.0 * eb_abs);
        q3.inv_hi = (float)q3.inv;
        q3.inv_lo = (float)(q3.inv - (double)q3.inv_hi);
        q3.slack = eb_abs * (1.0 + 1e-12);
        q3.r = (int32_t)(cap / 2);
        q3.cap = cap;
        q3.codes = codes;
        q3.hist = reinterpret_cast<unsigned long long *>(hist);
        q3.records = outliers;
        q3.out_capacity = outliers ? out_capacity : 0;
        q3.st = st;
        q3.lb = lb;
        q3.ticket = &tick[0];
        q3.nchunks = g.nbx * g.nby * g.nbz;
        q3.ntiles = (q3.nchunks + kQ3TileChunks - 1) / kQ3TileChunks;
        q3.slots = slots;
        q3.tile_cnt = tile_cnt;
        q3.over_list = over_list;
        q3.n_over = &tick[3];
        q3.tile_off = tile_off;
        const size_t esz = dtype == 0 ? 4 : 8;
        q3.vec_ok = (g.nx % (16 / esz) == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
        if (L.fast1d) q3.vec_ok = (reinterpret_cast<uintptr_t>(x) & 15) == 0;  // chunks start at 256 k
        size_t smem = (size_t)kQ3Warps * 2 * 32 * 16 * (dtype == 0 ? 4 : 8) +
                      (size_t)kQ3Warps * 512 * code_bytes + (size_t)kQ3Warps * 16 * 32 * 4 +
                      (size_t)cap * 4;
        const bool tma = L.fast3d && dtype == 0 && code_bytes == 2 && q3.vec_ok && (g.nbx % kT1Warps == 0) &&
                         tma_encode();
        if (tma) {
            T1Params tp;
            tp.q = q3;
            tp.tpr = (uint32_t)(g.nbx / kT1Warps);
            tp.nst = q3.nchunks / kT1Warps;
            CUtensorMap map;
            cuuint64_t dims[3] = {g.nx, g.ny, g.nz};
            cuuint64_t strides[2] = {g.nx * 4, g.nx * g.ny * 4};
            cuuint32_t box[3] = {32, 8, 8};
            cuuint32_t estr[3] = {1, 1, 1};
            if (tma_encode()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void *>(x), dims, strides, box,
                             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
                return LZB_E_CUDA;
            const size_t tsm = (size_t)kT1Stages * kT1Tile + 1024 + (size_t)kT1Warps * 16 * 32 * 4 +
                               (size_t)kT1Warps * 512 * 2 + (size_t)cap * 4;
            LZB_CUDA_TRY(set_dyn_smem(k_quantize3d8_tma, tsm));
            int per_sm = 0;
            LZB_CUDA_TRY(occupancy(&per_sm, k_quantize3d8_tma, kT1Threads, tsm));
            if (per_sm < 1) per_sm = 1;
            const uint64_t grid = umin64((uint64_t)device_sms() * per_sm, tp.nst);
            tp.step_q = (uint32_t)((grid ? grid : 1) / tp.tpr);
            tp.step_rem = (uint32_t)((grid ? grid : 1) % tp.tpr);
            k_quantize3d8_tma<<<(unsigned)(grid ? grid : 1), kT1Threads, tsm, s>>>(tp, map);
            LZB_LAUNCH_CHECK();
        }
        auto launch = [&](auto kern) -> int {
            LZB_CUDA_TRY(set_dyn_smem(kern, smem));
            int per_sm = 0;
            LZB_CUDA_TRY(occupancy(&per_sm, kern, kQ3Threads, smem));
            if (per_sm < 1) per_sm = 1;
            uint64_t grid = umin64((uint64_t)device_sms() * per_sm, (q3.ntiles + kQ3Warps - 1) / kQ3Warps);
            kern<<<(unsigned)(grid ? grid : 1), kQ3Threads, smem, s>>>(q3);
            LZB_LAUNCH_CHECK();
            return LZB_OK;
        };
        auto launch2d = [&](auto kern) -> int {
            const size_t sm2 = (size_t)kQ3Warps * 16 * 32 * 4 + (size_t)cap * 4;
            LZB_CUDA_TRY(set_dyn_smem(kern, sm2));
            int per_sm = 0;
            LZB_CUDA_TRY(occupancy(&per_sm, kern, kQ3Threads, sm2));
            if (per_sm < 1) per_sm = 1;
            uint64_t grid = umin64((uint64_t)device_sms() * per_sm, (q3.ntiles + kQ3Warps - 1) / kQ3Warps);
            kern<<<(unsigned)(grid ? grid : 1), kQ3Threads, sm2, s>>>(q3);
            LZB_LAUNCH_CHECK();
            return LZB_OK;
        };
        if (tma)
            rc = LZB_OK;
        else if (L.fast2d)
            rc = dtype == 0 ? (code_bytes == 2 ? launch2d(k_quantize_r8<2, float, uint16_t>)
                                               : launch2d(k_quantize_r8<2, float, uint32_t>))
                            : (code_bytes == 2 ? launch2d(k_quantize_r8<2, double, uint16_t>)
                                               : launch2d(k_quantize_r8<2, double, uint32_t>));
        else if (L.fast1d)
            rc = dtype == 0 ? (code_bytes == 2 ? launch2d(k_quantize_r8<1, float, uint16_t>)
                                               : launch2d(k_quantize_r8<1, float, uint32_t>))
                            : (code_bytes == 2 ? launch2d(k_quantize_r8<1, double, uint16_t>)
                                               : launch2d(k_quantize_r8<1, double, uint32_t>));
        else if (dtype == 0)
            rc = code_bytes == 2 ? launch(k_quantize3d8<float, uint16_t>) : launch(k_quantize3d8<float, uint32_t>);
        else
            rc = code_bytes == 2 ? launch(k_quantize3d8<double, uint16_t>) : launch(k_quantize3d8<double, uint32_t>);
        if (rc) return rc;
        if (hist_ev) LZB_CUDA_TRY(cudaEventRecord(hist_ev, s));  // the histogram is final
        // phase 2: tile offsets, slot compaction, overflow re-emission
        const int sms = device_sms();
        k_q3_scan<<<(unsigned)umin64((q3.ntiles + 2047) / 2048, (uint64_t)sms * 4), 256, 0, s>>>(
            q3, tile_off, slb, &tick[2]);
        LZB_LAUNCH_CHECK();
        if (outliers && out_capacity) {
            k_q3_compact<<<(unsigned)umin64((q3.ntiles * 32 + 255) / 256, (uint64_t)sms * 16), 256, 0, s>>>(q3);
            LZB_LAUNCH_CHECK();
            size_t esm = (size_t)kQ3Warps * 512 * code_bytes;
            if (L.fast2d || L.fast1d) {
                auto emit = [&](auto kern) { kern<<<sms, kQ3Threads, 0, s>>>(q3); };
                if (L.fast2d) {
                    if (dtype == 0) code_bytes == 2 ? emit(k_q2_emit<2, float, uint16_t>) : emit(k_q2_emit<2, float, uint32_t>);
                    else code_bytes == 2 ? emit(k_q2_emit<2, double, uint16_t>) : emit(k_q2_emit<2, double, uint32_t>);
                } else {
                    if (dtype == 0) code_bytes == 2 ? emit(k_q2_emit<1, float, uint16_t>) : emit(k_q2_emit<1, float, uint32_t>);
                    else code_bytes == 2 ? emit(k_q2_emit<1, double, uint16_t>) : emit(k_q2_emit<1, double, uint32_t>);
                }
            } else if (dtype == 0) {
                if (code_bytes == 2) k_q3_emit<float, uint16_t><<<sms, kQ3Threads, esm, s>>>(q3);
                else k_q3_emit<float, uint32_t><<<sms, kQ3Threads, esm, s>>>(q3);
            } else {
                if (code_bytes == 2) k_q3_emit<double, uint16_t><<<sms, kQ3Threads, esm, s>>>(q3);
                else k_q3_emit<double, uint32_t><<<sms, kQ3Threads, esm, s>>>(q3);
            }
            LZB_LAUNCH_CHECK();
        }
        LZB_CUDA_TRY(cudaMemsetAsync(&tick[2], 0, sizeof(unsigned int), s));  // reused below
        rc = LZB_OK;
        goto order;
    }
    if (dtype == 2) {
        if (L.box)
            rc = code_bytes == 2 ? launch_quant<int64_t, uint16_t, true>(qp, s)
                                 : launch_quant<int64_t, uint32_t, true>(qp, s);
        else
            rc = code_bytes == 2 ? launch_quant<int64_t, uint16_t, false>(qp, s)
                                 : launch_quant<int64_t, uint32_t, false>(qp, s);
    } else if (L.box) {
        if (dtype == 0)
            rc = code_bytes == 2 ? launch_quant<float, uint16_t, true>(qp, s)
                                 : launch_quant<float, uint32_t, true>(qp, s);
        else
            rc = code_bytes == 2 ? launch_quant<double, uint16_t, true>(qp, s)
                                 : launch_quant<double, uint32_t, true>(qp, s);
    } else {
        if (dtype == 0)
            rc = code_bytes == 2 ? launch_quant<float, uint16_t, false>(qp, s)
                                 : launch_quant<float, uint32_t, false>(qp, s);
        else
            rc = code_bytes == 2 ? launch_quant<double, uint16_t, false>(qp, s)
                                 : launch_quant<double, uint32_t, false>(qp, s);
    }
    if (rc) return rc;
    if (hist_ev) LZB_CUDA_TRY(cudaEventRecord(hist_ev, s));  // the histogram is final
order:
    if (!outliers || out_capacity == 0) return LZB_OK;

    // ---- global row-major ordering of the outlier records ----
    OrderParams op;
    op.records = outliers;
    op.tmp = tmp;
    op.st = st;
    op.capacity = out_capacity;
    op.g = g;
    op.unsorted = &tick[2];
    op.row_cnt = row_cnt;
    op.row_start = row_start;
    op.seg_start = seg_start;
    op.seg_end = seg_end;
    op.scan_lb = scan_lb;
    op.scan_ticket = &tick[1];
    const int sms = device_sms();
    k_check_sorted<<<sms * 4, 256, 0, s>>>(op);
    LZB_LAUNCH_CHECK();
    // the remaining launches exit immediately unless *unsorted was set
    LZB_CUDA_TRY(cudaMemsetAsync(row_cnt, 0, L.nrows_grid * sizeof(uint32_t), s));
    LZB_CUDA_TRY(cudaMemsetAsync(seg_end, 0, L.nrows_chunk * sizeof(uint64_t), s));
    LZB_CUDA_TRY(cudaMemsetAsync(scan_lb, 0, ((L.nrows_grid + 2047) / 2048 + 1) * sizeof(uint64_t), s));
    k_order_prepare<<<sms * 4, 256, 0, s>>>(op);
    LZB_LAUNCH_CHECK();
    uint64_t scan_tiles = (L.nrows_grid + 2047) / 2048;
    k_scan_u32<<<(unsigned)scan_tiles, 256, 0, s>>>(row_cnt, row_start, L.nrows_grid, scan_lb,
                                                   &tick[1], op.unsorted);
    LZB_LAUNCH_CHECK();
    uint64_t grid = L.nrows_chunk < (uint64_t)sms * 8 ? L.nrows_chunk : (uint64_t)sms * 8;
    k_order_scatter<<<(unsigned)(grid ? grid : 1), 256, 0, s>>>(op);
    LZB_LAUNCH_CHECK();
    return LZB_OK;
}

// ----------------------------------------------------------------------------
// Stand-alone prequantization (stage API, P/quantize.py:95-110)
// ----------------------------------------------------------------------------
template <typename InT>
__global__ void k_prequant(const InT *x, uint64_t n, double two_eb, double slack, int64_t *out,
                           lzb_dstatus *st) {
    int flags = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = prequant((double)x[i], two_eb, slack, flags);
    flags = __reduce_or_sync(0xffffffffu, flags);
    if (lane_id() == 0 && flags) set_status(st, (flags & 1) ? LZB_E_OVERFLOW : LZB_E_ASSERT);
}

extern "C" int lzb_prequantize(const void *x, int dtype, uint64_t n, double eb_abs, int64_t *out,
                               lzb_dstatus *st, void *stream) {
    if (!x || !out || !st || (dtype != 0 && dtype != 1)) return LZB_E_ARG;
    cudaStream_t s = as_stream(stream);
    LZB_CUDA_TRY(cudaMemsetAsync(st, 0, sizeof(lzb_dstatus), s));
    if (n == 0) return LZB_OK;
    unsigned grid = (unsigned)umin64((n + 255) / 256, (uint64_t)device_sms() * 16);
    if (dtype == 0)
        k_prequant<float><<<grid, 256, 0, s>>>((const float *)x, n, 2.0 * eb_abs,
                                               eb_abs * (1.0 + 1e-12), out, st);
    else
        k_prequant<double><<<grid, 256, 0, s>>>((const double *)x, n, 2.0 * eb_abs,
                                                eb_abs * (1.0 + 1e-12), out, st);
    LZB_LAUNCH_CHECK();
    return LZB_OK;
}

// ----------------------------------------------------------------------------
// Verification of K1's fast prequantizers against the exact reference rule
// (P/quantize.py:95-110): f32 inputs exhaustively by bit pattern range, f64
// inputs on hashed bit patterns.  A fast result that is ACCEPTED must equal
// the exact one (value, and no overflow / assert flag); rejected inputs take
// the exact path in K1, so they cannot disagree.
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint64_t pq_mix(uint64_t z) {  // splitmix64
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void k_pq_verify(uint64_t lo, uint64_t count, int dtype, double two_eb, double slack, double inv,
                            float inv_hi, float inv_lo, unsigned long long *cnt) {
    unsigned long long bad = 0, fast = 0, finite = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        double v;
        bool ok = true;
        int64_t f;
        if (dtype == 0) {
            const float x = __uint_as_float((uint32_t)(lo + i));
            if (!isfinite(x)) continue;
            f = f3::pq_fast_f32(x, inv_hi, inv_lo, ok);
            v = (double)x;
        } else {
            v = __longlong_as_double((long long)pq_mix(lo + i));
            if (!isfinite(v)) continue;
            f = f3::pq_fast(v, inv, ok);
        }
        finite++;
        if (!ok) continue;
        fast++;
        int flags = 0;
        const int64_t e = prequant(v, two_eb, slack, flags);
        if (flags || e != f) bad++;
    }
    bad = __reduce_add_sync(0xffffffffu, (unsigned)bad);
    fast = __reduce_add_sync(0xffffffffu, (unsigned)fast);
    finite = __reduce_add_sync(0xffffffffu, (unsigned)finite);
    if (lane_id() == 0) {
        if (bad) atomicAdd(&cnt[0], bad);
        atomicAdd(&cnt[1], fast);
        atomicAdd(&cnt[2], finite);
    }
}

extern "C" int lzb_prequant_verify(double eb_abs, uint64_t lo, uint64_t count, int dtype, lzb_dstatus *st,
                                   void *stream) {
    if (!st || (dtype != 0 && dtype != 1) || !(eb_abs > 0)) return LZB_E_ARG;
    cudaStream_t s = as_stream(stream);
    LZB_CUDA_TRY(cudaMemsetAsync(st, 0, sizeof(lzb_dstatus), s));
    if (count == 0) return LZB_OK;
    const double inv = 1.0 / (2.0 * eb_abs);  // exactly as lzb_quantize derives it
    const float inv_hi = (float)inv, inv_lo = (float)(inv - (double)inv_hi);
    unsigned grid = (unsigned)umin64((count + 255) / 256, (uint64_t)device_sms() * 32);
    k_pq_verify<<<grid, 256, 0, s>>>(lo, count, dtype, 2.0 * eb_abs, eb_abs * (1.0 + 1e-12), inv, inv_hi,
                                     inv_lo, reinterpret_cast<unsigned long long *>(st->u));
    LZB_LAUNCH_CHECK();
    return LZB_OK;
}

// ----------------------------------------------------------------------------
// Grid <-> chunk-major reorder (P/pipeline.py:102-117)
// ----------------------------------------------------------------------------
template <typename T>
__global__ void k_chunk_major(const T *src, T *dst, Geom g, int direction) {
    const uint64_t n = g.nx * g.ny * g.nz;
    for (uint64_t pos = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; pos < n;
         pos += (uint64_t)gridDim.x * blockDim.x) {
        StreamCoord c = stream_coord(g, pos);
        uint64_t gi = c.x + g.nx * (c.y + g.ny * c.z);
        if (direction == 0)
            dst[pos] = src[gi];
        else
            dst[gi] = src[pos];
    }
}

extern "C" int lzb_chunk_major(const void *src, void *dst, int elem_bytes, const lzb_geom *gg,
                               int direction, void *stream) {
    if (!src || !dst || !gg || (direction != 0 && direction != 1)) return LZB_E_ARG;
    Geom g = make_geom(*gg);
    uint64_t n = g.nx * g.ny * g.nz;
    cudaStream_t s = as_stream(stream);
    unsigned grid = (unsigned)umin64((n + 255) / 256, (uint64_t)device_sms() * 16);
    if (elem_bytes == 2)
        k_chunk_major<uint16_t><<<grid, 256, 0, s>>>((const uint16_t *)src, (uint16_t *)dst, g, direction);
    else if (elem_bytes == 4)
        k_chunk_major<uint32_t><<<grid, 256, 0, s>>>((const uint32_t *)src, (uint32_t *)dst, g, direction);
    else if (elem_bytes == 8)
        k_chunk_major<uint64_t><<<grid, 256, 0, s>>>((const uint64_t *)src, (uint64_t *)dst, g, direction);
    else
        return LZB_E_ARG;
    LZB_LAUNCH_CHECK();
    return LZB_OK;
}
