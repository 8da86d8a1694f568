// Histogram and K2: canonical Huffman code book on device.
//
// Reference semantics (P = /root/reference/pkg/src/lzebc):
//   histogram          P/codebook.py:23-27
//   _huffman_lengths   P/codebook.py:143-176  heap keyed (freq, tie); tie =
//                      symbol for leaves, cap + k for the k-th internal node
//   _canonical_codes   P/codebook.py:179-190  by ascending (length, symbol)
//   from_lengths       P/codebook.py:125-140  (Kraft validation)
//   average_bits       P/codebook.py:110-115  (selection rule input)
//
// K2 replaces the heap with the two-queue construction: leaves sorted by
// (freq, symbol) and internal nodes (created in non-decreasing weight order)
// popped by smallest weight, leaf first on ties.  Both keys are unique and the
// internal queue is ordered by (weight, creation), so the pop sequence -- and
// therefore the tree and every code length -- is identical to the reference's
// heapq sequence (pinned by tests/test_oracle_golden.py random_lengths and the
// -m gpu codebook parity test).
#include "lzb_common.cuh"

namespace lzb {

constexpr uint32_t kHistSmemMax = 4096;
constexpr int kCbThreads = 1024;
constexpr uint32_t kMaxCap = 1u << 20;

template <typename SymT>
__global__ void __launch_bounds__(256) k_histogram(const SymT *sym, uint64_t n, uint32_t cap,
                                                   unsigned long long *hist, lzb_dstatus *st) {
    extern __shared__ uint32_t s_h[];
    const bool sm = cap <= kHistSmemMax;
    if (sm)
        for (uint32_t i = threadIdx.x; i < cap; i += blockDim.x) s_h[i] = 0;
    __syncthreads();
    uint32_t bad = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t v = (uint32_t)sym[i];
        if (v >= cap) {
            bad = 1;
            continue;
        }
        if (sm)
            atomicAdd(&s_h[v], 1u);
        else
            atomicAdd(&hist[v], 1ull);
    }
    __syncthreads();
    if (sm)
        for (uint32_t i = threadIdx.x; i < cap; i += blockDim.x)
            if (s_h[i]) atomicAdd(&hist[i], (unsigned long long)s_h[i]);
    if (__any_sync(0xffffffffu, bad) && lane_id() == 0) set_status(st, LZB_E_DATA);
}

// ---------------------------------------------------------------------------
// K2: one CTA.
// ---------------------------------------------------------------------------
struct CbScratch {
    uint64_t *key;     // pow2 >= cap: (freq << 20) | symbol, sorted ascending
    uint64_t *wint;    // internal node weights
    uint32_t *parent;  // 2n-1 parents
    uint8_t *depth;    // 2n-1 depths
};

__device__ void bitonic_sort_u64(uint64_t *a, uint32_t n) {  // n power of two, block-wide
    for (uint32_t k = 2; k <= n; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
                uint32_t ixj = i ^ j;
                if (ixj > i) {
                    uint64_t x = a[i], y = a[ixj];
                    bool up = (i & k) == 0;
                    if ((x > y) == up) {
                        a[i] = y;
                        a[ixj] = x;
                    }
                }
            }
            __syncthreads();
        }
    }
}

// Canonical code words from lengths (P/codebook.py:179-190) + Kraft check
// (P/codebook.py:125-140).  Block-wide; returns a LZB code (0 ok).
__device__ int canonical_from_lengths(const uint8_t *lengths, uint32_t cap, uint64_t *codes,
                                      uint32_t *s_cnt /*65*/, uint64_t *s_first /*66*/,
                                      uint32_t *s_misc /*4*/, bool validate) {
    for (uint32_t i = threadIdx.x; i < 65; i += blockDim.x) s_cnt[i] = 0;
    if (threadIdx.x < 4) s_misc[threadIdx.x] = 0;
    __syncthreads();
    for (uint32_t s0 = 0; s0 < cap; s0 += blockDim.x) {  // warp-aggregated length counts
        const uint32_t s = s0 + threadIdx.x;
        const uint32_t L = s < cap ? lengths[s] : 0u;
        if (L > 64) atomicOr(&s_misc[0], 1u);
        const uint32_t Lc = L > 64 ? 0u : L;
        const uint32_t peers = __match_any_sync(0xffffffffu, Lc);
        if (Lc && (threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1)) atomicAdd(&s_cnt[Lc], (uint32_t)__popc(peers));
        const uint32_t wmax = __reduce_max_sync(0xffffffffu, Lc);
        if ((threadIdx.x & 31) == 0 && wmax) atomicMax(&s_misc[1], wmax);
    }
    __syncthreads();
    __shared__ int s_rc;
    if (threadIdx.x == 0) {
        int rc = 0;
        uint32_t used = 0;
        for (int L = 1; L <= 64; L++) used += s_cnt[L];
        s_misc[2] = used;
        if (s_misc[0]) rc = LZB_E_CORRUPT;  // "codebook length exceeds 64 bits"
        else if (used == 0) rc = LZB_E_CORRUPT;  // "codebook has no symbols"
        else if (used == 1) {
            if (validate && s_misc[1] != 1) rc = LZB_E_CORRUPT;  // single symbol must be length 1
        } else if (validate) {
            // Kraft equality: avail(L) = 2*avail(L-1) - cnt[L], must end at 0
            int64_t avail = 1;
            for (int L = 1; L <= 64 && !rc; L++) {
                avail = 2 * avail - (int64_t)s_cnt[L];
                if (avail < 0 || avail > (int64_t)cap) rc = LZB_E_CORRUPT;
            }
            if (!rc && avail != 0) rc = LZB_E_CORRUPT;
        }
        // first code per length: first[L] = (first[L-1] + cnt[L-1]) << 1
        uint64_t f = 0;
        s_first[0] = 0;
        for (int L = 1; L <= 64; L++) {
            f = (f + s_cnt[L - 1]) << 1;
            if (L == 1) f = 0;
            s_first[L] = f;
        }
        s_rc = rc;
    }
    __syncthreads();
    if (s_rc) return s_rc;
    // code = first[L] + rank of the symbol among equal lengths (ascending
    // symbol).  Warp 0 walks the symbols 32 at a time; peers with the same
    // length are ranked with match_any, s_first[] is the running counter.
    if (threadIdx.x < 32) {
        const uint32_t lane = threadIdx.x;
        for (uint32_t s0 = 0; s0 < cap; s0 += 32) {
            uint32_t s = s0 + lane;
            uint32_t L = s < cap ? lengths[s] : 0u;
            uint32_t peers = __match_any_sync(0xffffffffu, L);
            uint32_t rank = __popc(peers & ((1u << lane) - 1u));
            uint64_t base = s_first[L];
            if (s < cap) codes[s] = L ? base + rank : 0;
            __syncwarp();
            if (L && lane == (uint32_t)(__ffs(peers) - 1)) s_first[L] = base + __popc(peers);
            __syncwarp();
        }
    }
    __syncthreads();
    return 0;
}

__global__ void __launch_bounds__(kCbThreads) k_codebook(const unsigned long long *hist, uint32_t cap,
                                                        uint8_t *lengths, uint64_t *codes,
                                                        lzb_dstatus *st, CbScratch sc, uint32_t npow2,
                                                        int use_smem) {
    extern __shared__ __align__(16) unsigned char cb_smem[];
    if (use_smem) {  // small books: the whole tree lives in shared memory
        sc.key = reinterpret_cast<uint64_t *>(cb_smem);
        sc.wint = sc.key + npow2;
        sc.parent = reinterpret_cast<uint32_t *>(sc.wint + cap);
        sc.depth = reinterpret_cast<uint8_t *>(sc.parent + 2 * cap);
    }
    __shared__ uint32_t s_n;
    __shared__ uint32_t s_cnt[65];
    __shared__ uint64_t s_first[66];
    __shared__ uint32_t s_misc[4];
    __shared__ unsigned long long s_sum, s_tot;
    __shared__ int s_err;
    if (threadIdx.x == 0) {
        s_n = 0;
        s_sum = 0;
        s_tot = 0;
        s_err = 0;
    }
    __syncthreads();
    // compact nonzero symbols into sortable keys
    for (uint32_t s = threadIdx.x; s < npow2; s += blockDim.x) sc.key[s] = ~0ull;
    __syncthreads();
    for (uint32_t s0 = 0; s0 < cap; s0 += blockDim.x) {  // warp-aggregated compaction
        const uint32_t s = s0 + threadIdx.x;
        const uint64_t f = s < cap ? hist[s] : 0ull;
        if (s < cap) lengths[s] = 0;
        if (f >= (1ull << 44)) s_err = 1;
        const uint32_t m = __ballot_sync(0xffffffffu, f != 0);
        uint32_t k0 = 0;
        if ((threadIdx.x & 31) == 0 && m) k0 = atomicAdd(&s_n, (uint32_t)__popc(m));
        k0 = __shfl_sync(0xffffffffu, k0, 0);
        if (f) sc.key[k0 + __popc(m & ((1u << (threadIdx.x & 31)) - 1u))] = (f << 20) | s;
    }
    __syncthreads();
    const uint32_t n = s_n;
    if (n == 0 || s_err) {
        if (threadIdx.x == 0) set_status(st, LZB_E_DATA);  // empty histogram
        return;
    }
    bitonic_sort_u64(sc.key, npow2);
    if (n == 1) {
        if (threadIdx.x == 0) lengths[sc.key[0] & 0xFFFFF] = 1;  // lone symbol -> 1 bit
    } else {
        // two-queue Huffman merge (sequential; n-1 steps); the heads of both
        // queues are kept in registers
        if (threadIdx.x == 0) {
            uint32_t li = 0, ii = 0, ni = 0;
            uint64_t lw = sc.key[0] >> 20;  // head leaf weight (li < n)
            uint64_t iw = 0;                // head internal weight (ii < ni)
            for (uint32_t k = 0; k < n - 1; k++) {
                uint64_t w[2];
                uint32_t id[2];
#pragma unroll
                for (int t = 0; t < 2; t++) {
                    const bool take_leaf = li < n && (ii >= ni || lw <= iw);  // leaf first on ties
                    if (take_leaf) {
                        w[t] = lw;
                        id[t] = li++;
                        lw = li < n ? (sc.key[li] >> 20) : 0;
                    } else {
                        w[t] = iw;
                        id[t] = n + ii++;
                        iw = ii < ni ? sc.wint[ii] : 0;
                    }
                }
                const uint64_t nw = w[0] + w[1];
                sc.wint[ni] = nw;
                if (ii == ni) iw = nw;  // the queue was empty: the new node is its head
                sc.parent[id[0]] = n + ni;
                sc.parent[id[1]] = n + ni;
                ni++;
            }
        }
        __syncthreads();
        // depths (number of ancestors) of the 2n-1 nodes, root = node 2n-2
        const uint32_t nn = 2 * n - 1, root = nn - 1;
        if (nn <= 4 * blockDim.x) {  // pointer jumping: ceil(log2(nn)) rounds
            uint32_t *anc = sc.parent;  // reused as the jump pointers
            for (uint32_t i = threadIdx.x; i < nn; i += blockDim.x) sc.depth[i] = i == root ? 0 : 1;
            if (threadIdx.x == 0) anc[root] = root;
            __syncthreads();
            for (uint32_t span = 1; span < nn; span <<= 1) {
                uint32_t a_new[4], d_new[4];
#pragma unroll
                for (uint32_t c = 0; c < 4; c++) {
                    const uint32_t i = threadIdx.x + c * blockDim.x;
                    if (i < nn) {
                        const uint32_t a = anc[i];
                        d_new[c] = sc.depth[i] + sc.depth[a];
                        a_new[c] = anc[a];
                    }
                }
                __syncthreads();
#pragma unroll
                for (uint32_t c = 0; c < 4; c++) {
                    const uint32_t i = threadIdx.x + c * blockDim.x;
                    if (i < nn) {
                        sc.depth[i] = (uint8_t)(d_new[c] > 255 ? 255 : d_new[c]);
                        anc[i] = a_new[c];
                    }
                }
                __syncthreads();
            }
        } else {  // large books: top-down walk over the internal nodes
            if (threadIdx.x == 0) {
                sc.depth[root] = 0;
                for (int32_t k = (int32_t)root - 1; k >= (int32_t)n; k--) {
                    const uint32_t d = sc.depth[sc.parent[k]] + 1u;
                    sc.depth[k] = (uint8_t)(d > 255 ? 255 : d);
                }
            }
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
                const uint32_t d = sc.depth[sc.parent[i]] + 1u;
                sc.depth[i] = (uint8_t)(d > 255 ? 255 : d);
            }
            __syncthreads();
        }
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
            uint32_t d = sc.depth[i];
            if (d > 64) {
                s_err = 1;
                d = 64;
            }
            lengths[sc.key[i] & 0xFFFFF] = (uint8_t)d;
        }
    }
    __syncthreads();
    if (s_err) {
        if (threadIdx.x == 0) set_status(st, LZB_E_DATA);  // code longer than 64 bits
        return;
    }
    int rc = canonical_from_lengths(lengths, cap, codes, s_cnt, s_first, s_misc, false);
    if (rc) {
        if (threadIdx.x == 0) set_status(st, LZB_E_DATA);
        return;
    }
    // exact <b> inputs: sum(count * len) and total
    unsigned long long sum = 0, tot = 0;
    for (uint32_t s = threadIdx.x; s < cap; s += blockDim.x) {
        uint64_t f = hist[s];
        sum += f * lengths[s];
        tot += f;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {  // warp sums first: 32 shared atomics, not 1024
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
        tot += __shfl_xor_sync(0xffffffffu, tot, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&s_sum, sum);
        atomicAdd(&s_tot, tot);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        st->u[0] = s_sum;
        st->u[1] = s_tot;
        st->u[2] = s_misc[1];
        st->u[3] = n;
    }
}

__global__ void __launch_bounds__(kCbThreads) k_from_lengths(const uint8_t *lengths, uint32_t cap,
                                                            uint64_t *codes, lzb_dstatus *st) {
    __shared__ uint32_t s_cnt[65];
    __shared__ uint64_t s_first[66];
    __shared__ uint32_t s_misc[4];
    int rc = canonical_from_lengths(lengths, cap, codes, s_cnt, s_first, s_misc, true);
    if (threadIdx.x == 0) {
        if (rc) set_status(st, rc);
        st->u[2] = s_misc[1];
        st->u[3] = s_misc[2];
    }
}

static uint32_t pow2_at_least(uint32_t v) {
    uint32_t p = 1;
    while (p < v) p <<= 1;
    return p;
}

template <typename S>
static void cb_scratch(S &s, uint32_t cap) {
    uint32_t np = pow2_at_least(cap);
    s.template take<uint64_t>(np);
    s.template take<uint64_t>(cap);
    s.template take<uint32_t>(2 * cap);
    s.template take<uint8_t>(2 * cap);
}

}  // namespace lzb

using namespace lzb;

extern "C" int lzb_histogram(const void *sym, int sym_bytes, uint64_t n, uint32_t cap, uint64_t *hist,
                             lzb_dstatus *st, void *stream) {
    if (!hist || !st || (sym_bytes != 2 && sym_bytes != 4) || cap == 0) return LZB_E_ARG;
    cudaStream_t s = as_stream(stream);
    LZB_CUDA_TRY(cudaMemsetAsync(st, 0, sizeof(lzb_dstatus), s));
    LZB_CUDA_TRY(cudaMemsetAsync(hist, 0, cap * sizeof(uint64_t), s));
    if (n == 0) return LZB_OK;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    unsigned grid = (unsigned)umin64((n + 255) / 256, (uint64_t)sms * 8);
    size_t smem = cap <= kHistSmemMax ? cap * sizeof(uint32_t) : 0;
    if (sym_bytes == 2)
        k_histogram<uint16_t><<<grid, 256, smem, s>>>((const uint16_t *)sym, n, cap,
                                                      (unsigned long long *)hist, st);
    else
        k_histogram<uint32_t><<<grid, 256, smem, s>>>((const uint32_t *)sym, n, cap,
                                                      (unsigned long long *)hist, st);
    LZB_LAUNCH_CHECK();
    return LZB_OK;
}

extern "C" size_t lzb_codebook_scratch_bytes(uint32_t cap) {
    ScratchSize s;
    cb_scratch(s, cap);
    return s.bytes();
}

extern "C" int lzb_codebook(const uint64_t *hist, uint32_t cap, uint8_t *lengths, uint64_t *codes,
                            lzb_dstatus *st, void *scratch, size_t scratch_bytes, void *stream) {
    if (!hist || !lengths || !codes || !st || cap == 0 || cap > kMaxCap) return LZB_E_ARG;
    cudaStream_t s = as_stream(stream);
    Scratch sc(scratch, scratch_bytes);
    CbScratch c;
    uint32_t np = pow2_at_least(cap);
    c.key = sc.take<uint64_t>(np);
    c.wint = sc.take<uint64_t>(cap);
    c.parent = sc.take<uint32_t>(2 * cap);
    c.depth = sc.take<uint8_t>(2 * cap);
    if (!c.depth) return LZB_E_ARG;
    LZB_CUDA_TRY(cudaMemsetAsync(st, 0, sizeof(lzb_dstatus), s));
    size_t smem = (size_t)np * 8 + (size_t)cap * 8 + (size_t)cap * 8 + (size_t)cap * 2;
    int use_smem = smem <= 160 * 1024;
    if (use_smem)
        LZB_CUDA_TRY(cudaFuncSetAttribute(k_codebook, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
    k_codebook<<<1, kCbThreads, use_smem ? smem : 0, s>>>((const unsigned long long *)hist, cap,
                                                          lengths, codes, st, c, np, use_smem);
    LZB_LAUNCH_CHECK();
    return LZB_OK;
}

extern "C" int lzb_codebook_from_lengths(const uint8_t *lengths, uint32_t cap, uint64_t *codes,
                                         lzb_dstatus *st, void *scratch, size_t scratch_bytes,
                                         void *stream) {
    (void)scratch;
    (void)scratch_bytes;
    if (!lengths || !codes || !st || cap == 0) return LZB_E_ARG;
    cudaStream_t s = as_stream(stream);
    LZB_CUDA_TRY(cudaMemsetAsync(st, 0, sizeof(lzb_dstatus), s));
    k_from_lengths<<<1, kCbThreads, 0, s>>>(lengths, cap, codes, st);
    LZB_LAUNCH_CHECK();
    return LZB_OK;
}
