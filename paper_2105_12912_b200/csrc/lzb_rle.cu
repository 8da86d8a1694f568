// K4 run-length encode and K7 run-length decode.
//
// Reference semantics (P = /root/reference/pkg/src/lzebc):
//   run_length_encode  P/rle.py:17-35  maximal runs, u32 values and lengths;
//                      a run longer than _MAX_RUN (0xFFFFFFFF) becomes
//                      ceil(L/MAX) runs, all MAX long except the last
//   run_length_decode  P/rle.py:38-44  + the archive checks of
//                      P/pipeline.py:283-302 (section sizes, sum == count,
//                      symbol < cap), validated BEFORE expanding
//
// K4: one pass -- run heads flagged against the previous symbol,
// block scan + decoupled look-back give each head its run index; the head
// writes (value, start).  Lengths are adjacent start differences.  Splitting
// of over-long runs (only possible when n > max_run) runs as a scan + scatter
// pass that is skipped on device when no run exceeds max_run.
// K7: lengths scanned to u64 run starts (look-back), validated, then every
// 4096-symbol output tile binary-searches its first run and expands.
#include "lzb_common.cuh"

namespace lzb {

constexpr int kRThreads = 256;
constexpr int kRItems = 16;
constexpr int kRTile = kRThreads * kRItems;

template <typename SymT>
__global__ void __launch_bounds__(kRThreads) k_rle_heads(const SymT *sym, uint64_t n, uint32_t *vals,
                                                         uint64_t *starts, uint64_t cap_runs,
                                                         uint64_t *lb, unsigned int *ticket,
                                                         uint64_t ntiles, lzb_dstatus *st) {
    __shared__ uint32_t s_scan[33];
    __shared__ uint64_t s_tile, s_ex;
    while (true) {
        if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
        __syncthreads();
        const uint64_t t = s_tile;
        if (t >= ntiles) break;
        const uint64_t base = t * kRTile + (uint64_t)threadIdx.x * kRItems;
        uint32_t v[kRItems];
        uint32_t prev = base > 0 && base - 1 < n ? (uint32_t)sym[base - 1] : 0xFFFFFFFFu;
        uint32_t heads = 0, cnt = 0;
#pragma unroll
        for (int k = 0; k < kRItems; k++) {
            bool in = base + k < n;
            v[k] = in ? (uint32_t)sym[base + k] : 0u;
            bool h = in && (base + k == 0 || v[k] != prev);
            heads |= (uint32_t)h << k;
            cnt += h;
            prev = v[k];
        }
        uint32_t total;
        uint32_t off = block_exclusive_scan<uint32_t>(cnt, s_scan, &total);
        if ((threadIdx.x >> 5) == 0) {
            uint64_t ex = lookback_warp(lb, t, total);
            if (lane_id() == 0) s_ex = ex;
        }
        __syncthreads();
        uint64_t r = s_ex + off;
#pragma unroll
        for (int k = 0; k < kRItems; k++) {
            if ((heads >> k) & 1u) {
                if (r < cap_runs) {
                    vals[r] = v[k];
                    starts[r] = base + k;
                }
                r++;
            }
        }
        if (t == ntiles - 1 && threadIdx.x == 0) st->u[1] = s_ex + total;  // maximal runs
        __syncthreads();
    }
}

// lengths from adjacent starts; flags any run longer than max_run
__global__ void k_rle_lengths(const uint64_t *starts, uint64_t n, uint64_t cap_runs, uint64_t max_run,
                              uint64_t *len64, unsigned int *needs_split, lzb_dstatus *st) {
    const uint64_t R = st->u[1];
    if (R > cap_runs) return;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < R;
         r += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t e = r + 1 < R ? starts[r + 1] : n;
        uint64_t L = e - starts[r];
        len64[r] = L;
        if (L > max_run) *needs_split = 1u;
    }
}

// no split: final arrays directly; split: pieces per run
__global__ void k_rle_emit(const uint32_t *vals, const uint64_t *len64, uint64_t cap_runs,
                           uint64_t max_run, const unsigned int *needs_split, uint32_t *out_vals,
                           uint32_t *out_lens, uint32_t *pieces, lzb_dstatus *st) {
    const uint64_t R = st->u[1];
    if (R > cap_runs) return;
    const bool split = *needs_split != 0;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < R;
         r += (uint64_t)gridDim.x * blockDim.x) {
        if (!split) {
            out_vals[r] = vals[r];
            out_lens[r] = (uint32_t)len64[r];
        } else {
            pieces[r] = (uint32_t)((len64[r] + max_run - 1) / max_run);
        }
    }
    if (!split && blockIdx.x == 0 && threadIdx.x == 0) st->u[0] = R;
}

// split path: scan pieces then scatter
__global__ void __launch_bounds__(256) k_rle_scan_pieces(const uint32_t *pieces, uint64_t *pos,
                                                         uint64_t *lb, unsigned int *ticket,
                                                         const unsigned int *needs_split,
                                                         lzb_dstatus *st, uint64_t cap_runs) {
    if (!*needs_split) return;
    const uint64_t R = st->u[1];
    if (R > cap_runs) return;
    __shared__ uint64_t s_t, s_ex;
    __shared__ uint64_t s_scan[33];
    const uint64_t ntiles = (R + 2047) / 2048;
    while (true) {
        if (threadIdx.x == 0) s_t = atomicAdd(ticket, 1u);
        __syncthreads();
        const uint64_t t = s_t;
        if (t >= ntiles) break;
        const uint64_t base = t * 2048 + threadIdx.x * 8;
        uint64_t v[8], sum = 0;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            v[k] = base + k < R ? pieces[base + k] : 0;
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
        for (int k = 0; k < 8; k++)
            if (base + k < R) {
                pos[base + k] = run;
                run += v[k];
            }
        if (t == ntiles - 1 && threadIdx.x == 0) st->u[0] = s_ex + tot;
        __syncthreads();
    }
}

__global__ void k_rle_split_scatter(const uint32_t *vals, const uint64_t *len64, const uint32_t *pieces,
                                    const uint64_t *pos, uint64_t max_run, uint64_t cap_out,
                                    const unsigned int *needs_split, uint32_t *out_vals,
                                    uint32_t *out_lens, lzb_dstatus *st, uint64_t cap_runs) {
    if (!*needs_split) return;
    const uint64_t R = st->u[1];
    if (R > cap_runs) return;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < R;
         r += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t p0 = pos[r], k = pieces[r], L = len64[r];
        for (uint64_t j = 0; j < k; j++) {
            if (p0 + j >= cap_out) break;
            out_vals[p0 + j] = vals[r];
            out_lens[p0 + j] = (uint32_t)(j + 1 < k ? max_run : L - (k - 1) * max_run);
        }
    }
}

__global__ void k_rle_capacity(lzb_dstatus *st, uint64_t cap_runs, uint64_t cap_out) {
    if (st->u[1] > cap_runs || st->u[0] > cap_out) set_status(st, LZB_E_CAPACITY);
}

// ---------------------------------------------------------------------------
// K7 decode
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t ld_le32(const uint8_t *p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

__global__ void __launch_bounds__(256) k_rld_scan(const uint8_t *vals_le, const uint8_t *lens_le,
                                                  uint64_t R, uint32_t cap, uint32_t *vals,
                                                  uint64_t *starts, uint64_t *lb,
                                                  unsigned int *ticket, lzb_dstatus *st) {
    __shared__ uint64_t s_t, s_ex;
    __shared__ uint64_t s_scan[33];
    const uint64_t ntiles = (R + 2047) / 2048;
    int bad = 0;
    while (true) {
        if (threadIdx.x == 0) s_t = atomicAdd(ticket, 1u);
        __syncthreads();
        const uint64_t t = s_t;
        if (t >= ntiles) break;
        const uint64_t base = t * 2048 + threadIdx.x * 8;
        uint64_t v[8], sum = 0;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            v[k] = 0;
            if (base + k < R) {
                v[k] = ld_le32(lens_le + 4 * (base + k));
                uint32_t val = ld_le32(vals_le + 4 * (base + k));
                if (v[k] == 0 || val >= cap) bad = 1;
                vals[base + k] = val;
            }
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
        for (int k = 0; k < 8; k++)
            if (base + k < R) {
                starts[base + k] = run;
                run += v[k];
            }
        if (t == ntiles - 1 && threadIdx.x == 0) st->u[0] = s_ex + tot;
        __syncthreads();
    }
    if (__any_sync(0xffffffffu, bad) && lane_id() == 0) set_status(st, LZB_E_CORRUPT);
}

__global__ void k_rld_check(lzb_dstatus *st, uint64_t n) {
    if (st->u[0] != n) set_status(st, LZB_E_CORRUPT);
}

template <typename SymT>
__global__ void k_rld_expand(const uint32_t *vals, const uint64_t *starts, uint64_t R, SymT *out,
                             uint64_t n, const lzb_dstatus *st) {
    if (st->code) return;
    const uint64_t ntiles = (n + 4095) / 4096;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint64_t p0 = t * 4096, p1 = umin64(p0 + 4096, n);
        __shared__ uint64_t s_r0;
        if (threadIdx.x == 0) {  // last run with start <= p0
            uint64_t lo = 0, hi = R - 1;
            while (lo < hi) {
                uint64_t mid = (lo + hi + 1) / 2;
                if (starts[mid] <= p0) lo = mid;
                else hi = mid - 1;
            }
            s_r0 = lo;
        }
        __syncthreads();
        uint64_t r = s_r0;
        // each thread walks forward from the tile's first run (runs are usually long)
        for (uint64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
            while (r + 1 < R && starts[r + 1] <= p) r++;
            out[p] = (SymT)vals[r];
        }
        __syncthreads();
    }
}

static int sms() {
    int dev = 0, s = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
    return s > 0 ? s : 148;
}

// Maximal-run count of a symbol stream (sizes K4's outputs).  Each thread
// compares 8 consecutive symbols (one 16-byte load for u16) with their
// predecessors; the block total goes to st->u[0] with one atomic.
template <typename SymT>
__global__ void __launch_bounds__(256) k_count_runs(const SymT *sym, uint64_t n, lzb_dstatus *st) {
    unsigned long long heads = 0;
    const uint64_t ngroups = (n + 7) / 8;
    for (uint64_t gidx = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; gidx < ngroups;
         gidx += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t b = gidx * 8;
        uint32_t prev = b > 0 ? (uint32_t)__ldg(sym + b - 1) : ~(uint32_t)sym[0];
        if (b + 8 <= n && sizeof(SymT) == 2 && (reinterpret_cast<uintptr_t>(sym + b) & 15) == 0) {
            uint4 v = __ldg(reinterpret_cast<const uint4 *>(sym + b));
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const uint32_t lo = w[k] & 0xFFFFu, hi = w[k] >> 16;
                heads += (lo != prev) + (hi != lo);
                prev = hi;
            }
        } else {
            const uint64_t e = b + 8 < n ? b + 8 : n;
            for (uint64_t i = b; i < e; i++) {
                const uint32_t c = (uint32_t)__ldg(sym + i);
                heads += c != prev;
                prev = c;
            }
        }
    }
    heads = __reduce_add_sync(0xffffffffu, (unsigned)heads);
    if (lane_id() == 0 && heads) atomicAdd(reinterpret_cast<unsigned long long *>(&st->u[0]), heads);
}

}  // namespace lzb

using namespace lzb;

extern "C" int lzb_count_runs(const void *sym, int sym_bytes, uint64_t n, lzb_dstatus *st,
                              void *stream) {
    if (!st || (n && !sym) || (sym_bytes != 2 && sym_bytes != 4)) return LZB_E_ARG;
    cudaStream_t s = as_stream(stream);
    LZB_CUDA_TRY(cudaMemsetAsync(st, 0, sizeof(lzb_dstatus), s));
    if (n == 0) return LZB_OK;
    const uint64_t ng = (n + 7) / 8;
    const unsigned grid = (unsigned)umin64((ng + 255) / 256, (uint64_t)sms() * 8);
    if (sym_bytes == 2) k_count_runs<uint16_t><<<grid, 256, 0, s>>>(static_cast<const uint16_t *>(sym), n, st);
    else k_count_runs<uint32_t><<<grid, 256, 0, s>>>(static_cast<const uint32_t *>(sym), n, st);
    LZB_LAUNCH_CHECK();
    return LZB_OK;
}

extern "C" size_t lzb_rle_encode_scratch_bytes(uint64_t n) {
    // cap_runs is bounded by n
    ScratchSize s;
    uint64_t nt = (n + kRTile - 1) / kRTile;
    s.take<uint64_t>(nt ? nt : 1);
    s.take<unsigned int>(8);
    s.take<uint32_t>(n ? n : 1);  // vals
    s.take<uint64_t>(n ? n : 1);  // starts
    s.take<uint64_t>(n ? n : 1);  // len64
    s.take<uint32_t>(n ? n : 1);  // pieces
    s.take<uint64_t>(n ? n : 1);  // pos
    s.take<uint64_t>((n + 2047) / 2048 + 1);
    return s.bytes();
}

// Scratch for a known run count (preferred: the host learns R from K1).
extern "C" size_t lzb_rle_encode_scratch_bytes_runs(uint64_t n, uint64_t cap_runs) {
    ScratchSize s;
    uint64_t nt = (n + kRTile - 1) / kRTile;
    uint64_t c = cap_runs ? cap_runs : 1;
    s.take<uint64_t>(nt ? nt : 1);
    s.take<unsigned int>(8);
    s.take<uint32_t>(c);
    s.take<uint64_t>(c);
    s.take<uint64_t>(c);
    s.take<uint32_t>(c);
    s.take<uint64_t>(c);
    s.take<uint64_t>((c + 2047) / 2048 + 1);
    return s.bytes();
}

extern "C" int lzb_rle_encode(const void *sym, int sym_bytes, uint64_t n, uint32_t *values,
                              uint32_t *lengths, uint64_t cap_runs, uint64_t max_run,
                              lzb_dstatus *st, void *scratch, size_t scratch_bytes, void *stream) {
    if (!st || (sym_bytes != 2 && sym_bytes != 4) || max_run == 0) return LZB_E_ARG;
    cudaStream_t s = as_stream(stream);
    LZB_CUDA_TRY(cudaMemsetAsync(st, 0, sizeof(lzb_dstatus), s));
    if (n == 0) return LZB_OK;
    if (!sym || !values || !lengths) return LZB_E_ARG;
    const uint64_t nt = (n + kRTile - 1) / kRTile;
    // internal arrays are sized by the maximal-run capacity; the output
    // capacity cap_runs also bounds the split pieces
    const uint64_t c = cap_runs;
    Scratch sc(scratch, scratch_bytes);
    uint64_t *lb = sc.take<uint64_t>(nt);
    unsigned int *tick = sc.take<unsigned int>(8);
    uint32_t *vals = sc.take<uint32_t>(c);
    uint64_t *starts = sc.take<uint64_t>(c);
    uint64_t *len64 = sc.take<uint64_t>(c);
    uint32_t *pieces = sc.take<uint32_t>(c);
    uint64_t *pos = sc.take<uint64_t>(c);
    uint64_t *lb2 = sc.take<uint64_t>((c + 2047) / 2048 + 1);
    if (!lb2) return LZB_E_ARG;
    LZB_CUDA_TRY(cudaMemsetAsync(lb, 0, nt * sizeof(uint64_t), s));
    LZB_CUDA_TRY(cudaMemsetAsync(tick, 0, 8 * sizeof(unsigned int), s));
    LZB_CUDA_TRY(cudaMemsetAsync(lb2, 0, ((c + 2047) / 2048 + 1) * sizeof(uint64_t), s));
    const int nsm = sms();
    unsigned grid = (unsigned)umin64(nt, (uint64_t)nsm * 8);
    if (sym_bytes == 2)
        k_rle_heads<uint16_t><<<grid, kRThreads, 0, s>>>((const uint16_t *)sym, n, vals, starts, c, lb,
                                                         &tick[0], nt, st);
    else
        k_rle_heads<uint32_t><<<grid, kRThreads, 0, s>>>((const uint32_t *)sym, n, vals, starts, c, lb,
                                                         &tick[0], nt, st);
    LZB_LAUNCH_CHECK();
    unsigned g2 = (unsigned)umin64((c + 255) / 256, (uint64_t)nsm * 16);
    k_rle_lengths<<<g2 ? g2 : 1, 256, 0, s>>>(starts, n, c, max_run, len64, &tick[2], st);
    LZB_LAUNCH_CHECK();
    k_rle_emit<<<g2 ? g2 : 1, 256, 0, s>>>(vals, len64, c, max_run, &tick[2], values, lengths, pieces, st);
    LZB_LAUNCH_CHECK();
    k_rle_scan_pieces<<<(unsigned)umin64((c + 2047) / 2048, (uint64_t)nsm * 4) + 0u, 256, 0, s>>>(
        pieces, pos, lb2, &tick[1], &tick[2], st, c);
    LZB_LAUNCH_CHECK();
    k_rle_split_scatter<<<g2 ? g2 : 1, 256, 0, s>>>(vals, len64, pieces, pos, max_run, cap_runs,
                                                    &tick[2], values, lengths, st, c);
    LZB_LAUNCH_CHECK();
    k_rle_capacity<<<1, 1, 0, s>>>(st, c, cap_runs);
    LZB_LAUNCH_CHECK();
    return LZB_OK;
}

extern "C" size_t lzb_rle_decode_scratch_bytes(uint64_t runs) {
    ScratchSize s;
    uint64_t r = runs ? runs : 1;
    s.take<uint32_t>(r);
    s.take<uint64_t>(r);
    s.take<uint64_t>((r + 2047) / 2048 + 1);
    s.take<unsigned int>(4);
    return s.bytes();
}

extern "C" int lzb_rle_decode(const uint8_t *values_le, const uint8_t *lengths_le, uint64_t runs,
                              uint32_t cap, void *sym, int sym_bytes, uint64_t n, lzb_dstatus *st,
                              void *scratch, size_t scratch_bytes, void *stream) {
    if (!st || (sym_bytes != 2 && sym_bytes != 4)) return LZB_E_ARG;
    cudaStream_t s = as_stream(stream);
    LZB_CUDA_TRY(cudaMemsetAsync(st, 0, sizeof(lzb_dstatus), s));
    if (runs == 0) {
        if (n != 0) {
            int32_t code = LZB_E_CORRUPT;
            LZB_CUDA_TRY(cudaMemcpyAsync(&st->code, &code, sizeof(code), cudaMemcpyHostToDevice, s));
            LZB_CUDA_TRY(cudaStreamSynchronize(s));
        }
        return LZB_OK;
    }
    if (!values_le || !lengths_le || !sym) return LZB_E_ARG;
    Scratch sc(scratch, scratch_bytes);
    uint32_t *vals = sc.take<uint32_t>(runs);
    uint64_t *starts = sc.take<uint64_t>(runs);
    uint64_t *lb = sc.take<uint64_t>((runs + 2047) / 2048 + 1);
    unsigned int *tick = sc.take<unsigned int>(4);
    if (!tick) return LZB_E_ARG;
    LZB_CUDA_TRY(cudaMemsetAsync(lb, 0, ((runs + 2047) / 2048 + 1) * sizeof(uint64_t), s));
    LZB_CUDA_TRY(cudaMemsetAsync(tick, 0, 4 * sizeof(unsigned int), s));
    const int nsm = sms();
    k_rld_scan<<<(unsigned)umin64((runs + 2047) / 2048, (uint64_t)nsm * 4), 256, 0, s>>>(
        values_le, lengths_le, runs, cap, vals, starts, lb, &tick[0], st);
    LZB_LAUNCH_CHECK();
    k_rld_check<<<1, 1, 0, s>>>(st, n);
    LZB_LAUNCH_CHECK();
    unsigned grid = (unsigned)umin64((n + 4095) / 4096, (uint64_t)nsm * 16);
    if (grid == 0) grid = 1;
    if (sym_bytes == 2)
        k_rld_expand<uint16_t><<<grid, 256, 0, s>>>(vals, starts, runs, (uint16_t *)sym, n, st);
    else
        k_rld_expand<uint32_t><<<grid, 256, 0, s>>>(vals, starts, runs, (uint32_t *)sym, n, st);
    LZB_LAUNCH_CHECK();
    return LZB_OK;
}
