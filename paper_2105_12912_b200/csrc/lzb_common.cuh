// Shared device helpers for liblzb (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <tuple>

#include "../../include/lzb.h"

#define LZB_CUDA_TRY(expr)                                         \
    do {                                                           \
        cudaError_t _e = (expr);                                   \
        if (_e != cudaSuccess) return LZB_E_CUDA;                  \
    } while (0)

#define LZB_LAUNCH_CHECK() LZB_CUDA_TRY(cudaGetLastError())

namespace lzb {

// Host-side launch configuration cache.  cudaFuncSetAttribute (dynamic
// shared memory opt-in) and the occupancy query cost microseconds per call,
// which a small field would pay on every launch; both are per (device,
// kernel[, block, shared memory]) constants, so they are asked once.
struct LaunchCache {
    std::mutex mu;
    std::map<std::tuple<int, const void *>, size_t> smem;
    std::map<std::tuple<int, const void *, int, size_t>, int> occ;
};
static inline LaunchCache &launch_cache() {
    static LaunchCache c;
    return c;
}
template <typename K>
static inline cudaError_t set_dyn_smem(K kern, size_t bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    LaunchCache &c = launch_cache();
    const auto key = std::make_tuple(dev, reinterpret_cast<const void *>(kern));
    std::lock_guard<std::mutex> g(c.mu);
    auto it = c.smem.find(key);
    if (it != c.smem.end() && it->second >= bytes) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) c.smem[key] = bytes;
    return e;
}
template <typename K>
static inline cudaError_t occupancy(int *per_sm, K kern, int threads, size_t smem) {
    int dev = 0;
    cudaGetDevice(&dev);
    LaunchCache &c = launch_cache();
    const auto key = std::make_tuple(dev, reinterpret_cast<const void *>(kern), threads, smem);
    std::lock_guard<std::mutex> g(c.mu);
    auto it = c.occ.find(key);
    if (it != c.occ.end()) {
        *per_sm = it->second;
        return cudaSuccess;
    }
    const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, kern, threads, smem);
    if (e == cudaSuccess) c.occ[key] = *per_sm;
    return e;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda);
// a cached function pointer, nullptr if the driver lacks it.
static PFN_cuTensorMapEncodeTiled_v12000 tma_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
        tried = true;
    }
    return fn;
}


constexpr int kNumSMs = 148;  // B200; launch sizes are re-derived from the device at runtime

static inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

static inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Bump allocator over caller-provided scratch.
struct Scratch {
    char *base;
    size_t size, used;
    Scratch(void *b, size_t s) : base(static_cast<char *>(b)), size(s), used(0) {}
    template <typename T>
    T *take(size_t count) {
        size_t off = align_up(used, 256);
        size_t need = off + count * sizeof(T);
        if (need > size) return nullptr;
        used = need;
        return reinterpret_cast<T *>(base + off);
    }
};

// Size-only twin of Scratch, used by the *_scratch_bytes queries.
struct ScratchSize {
    size_t used = 0;
    template <typename T>
    void take(size_t count) { used = align_up(used, 256) + count * sizeof(T); }
    size_t bytes() const { return align_up(used, 256) + 256; }
};

// First error wins.
__device__ __forceinline__ void set_status(lzb_dstatus *st, int code) {
    atomicCAS(&st->code, 0, code);
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ uint32_t bswap32(uint32_t v) { return __byte_perm(v, 0, 0x0123); }

// ----------------------------------------------------------------------------
// Decoupled look-back exclusive scan over tiles (single pass).
// Status word per tile: [2-bit flag | 62-bit value]; flag 1 = aggregate,
// 2 = inclusive prefix.  Tiles must be claimed in increasing order by a
// ticket (so every waited-on predecessor is resident or finished).
// ----------------------------------------------------------------------------
constexpr uint64_t kLbAgg = 1ull << 62;
constexpr uint64_t kLbInc = 2ull << 62;
constexpr uint64_t kLbMask = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t lb_load(const uint64_t *p) {
    return *reinterpret_cast<const volatile uint64_t *>(p);
}
__device__ __forceinline__ void lb_store(uint64_t *p, uint64_t v) {
    *reinterpret_cast<volatile uint64_t *>(p) = v;
}

// Called by ONE full warp.  Returns the exclusive prefix of `tile` (same value
// in every lane) and publishes the inclusive prefix.
__device__ __forceinline__ uint64_t lookback_warp(uint64_t *status, uint64_t tile, uint64_t agg) {
    const uint32_t lane = lane_id();
    if (tile == 0) {
        if (lane == 0) lb_store(&status[0], kLbInc | agg);
        return 0;
    }
    if (lane == 0) lb_store(&status[tile], kLbAgg | agg);
    uint64_t excl = 0;
    int64_t base = (int64_t)tile - 1;
    while (true) {
        int64_t idx = base - (int64_t)lane;
        uint64_t v = (idx >= 0) ? lb_load(&status[idx]) : (kLbInc | 0ull);
        while (__any_sync(0xffffffffu, (v >> 62) == 0)) {
            if ((v >> 62) == 0) v = lb_load(&status[idx]);
        }
        uint32_t inc = __ballot_sync(0xffffffffu, (v >> 62) == 2);
        uint64_t val = v & kLbMask;
        if (inc) {
            uint32_t first = __ffs(inc) - 1;  // closest predecessor with an inclusive prefix
            if (lane > first) val = 0;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
        excl += val;
        if (inc) break;
        base -= 32;
    }
    if (lane == 0) lb_store(&status[tile], kLbInc | (excl + agg));
    return excl;
}

// Split form for deferred resolution: publish the aggregate as soon as it is
// known, do other work, then resolve (by then predecessors have usually
// published, so the look-back rarely spins).
__device__ __forceinline__ void lb_publish(uint64_t *status, uint64_t tile, uint64_t agg) {
    if (lane_id() == 0) lb_store(&status[tile], (tile == 0 ? kLbInc : kLbAgg) | agg);
}

// Called by one full warp after lb_publish(tile, agg); returns the exclusive
// prefix and publishes the inclusive one.
__device__ __forceinline__ uint64_t lb_resolve(uint64_t *status, uint64_t tile, uint64_t agg) {
    const uint32_t lane = lane_id();
    if (tile == 0) return 0;
    uint64_t excl = 0;
    int64_t base = (int64_t)tile - 1;
    while (true) {
        int64_t idx = base - (int64_t)lane;
        uint64_t v = (idx >= 0) ? lb_load(&status[idx]) : (kLbInc | 0ull);
        while (__any_sync(0xffffffffu, (v >> 62) == 0)) {
            if ((v >> 62) == 0) v = lb_load(&status[idx]);
        }
        uint32_t inc = __ballot_sync(0xffffffffu, (v >> 62) == 2);
        uint64_t val = v & kLbMask;
        if (inc) {
            uint32_t first = __ffs(inc) - 1;
            if (lane > first) val = 0;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
        excl += val;
        if (inc) break;
        base -= 32;
    }
    if (lane == 0) lb_store(&status[tile], kLbInc | (excl + agg));
    return excl;
}

// Block-wide exclusive scan of one u32 per thread (blockDim multiple of 32,
// <= 1024).  `warp_sums` needs 33 entries of shared memory.  Returns the
// exclusive prefix; *total receives the block total.
template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T *warp_sums, T *total) {
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    const uint32_t nwarps = blockDim.x >> 5;
    T incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += t;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        T w = lane < nwarps ? warp_sums[lane] : T(0);
        T wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= (uint32_t)o) wi += t;
        }
        if (lane < nwarps) warp_sums[lane] = wi - w;
        if (lane == nwarps - 1) warp_sums[32] = wi;
    }
    __syncthreads();
    T res = warp_sums[warp] + incl - v;
    *total = warp_sums[32];
    __syncthreads();
    return res;
}

// Chunk-major addressing (P/pipeline.py:102-105):
// chunk (bx,by,bz) starts at nx*ny*cz*bz + nx*ez*cy*by + ez*ey*cx*bx.
struct Geom {
    uint64_t nx, ny, nz, cx, cy, cz;
    uint64_t nbx, nby, nbz;
    int ndim;
};

static inline Geom make_geom(const lzb_geom &g) {
    Geom r;
    r.nx = g.nx; r.ny = g.ny; r.nz = g.nz;
    r.cx = g.cx; r.cy = g.cy; r.cz = g.cz;
    r.nbx = (g.nx + g.cx - 1) / g.cx;
    r.nby = (g.ny + g.cy - 1) / g.cy;
    r.nbz = (g.nz + g.cz - 1) / g.cz;
    r.ndim = g.ndim;
    return r;
}

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

__host__ __device__ __forceinline__ uint64_t chunk_base(const Geom &g, uint64_t bx, uint64_t by,
                                                        uint64_t bz) {
    uint64_t ez = umin64(g.cz, g.nz - bz * g.cz);
    uint64_t ey = umin64(g.cy, g.ny - by * g.cy);
    return g.nx * g.ny * g.cz * bz + g.nx * ez * g.cy * by + ez * ey * g.cx * bx;
}

template <typename T>
__device__ __forceinline__ T load_sym(const void *p, uint64_t i);
template <>
__device__ __forceinline__ uint32_t load_sym<uint32_t>(const void *p, uint64_t i) {
    return static_cast<const uint32_t *>(p)[i];
}

}  // namespace lzb
