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

// Ascending sort of np (a power of two) keys a[0..np) with one CTA: 32-key
// runs sorted in registers per warp (bitonic over shuffles), then
// log2(np/32) merge levels where every key finds its place by a binary
// search in the partner run (ties -- the ~0 padding -- resolved left run
// first, so every slot is written once).  Ping-pongs between
// a and b; returns the buffer holding the result.  About a dozen block
// barriers instead of the bitonic network's 55.
__device__ uint64_t *sort_u64_merge(uint64_t *a, uint64_t *b, uint32_t np, uint32_t nbuf) {
    const uint32_t lane = threadIdx.x & 31u;
    for (uint32_t i0 = threadIdx.x & ~31u; i0 < np; i0 += blockDim.x) {
        const uint32_t i = i0 + lane;
        uint64_t v = i < nbuf ? a[i] : ~0ull;
#pragma unroll
        for (uint32_t k = 2; k <= 32; k <<= 1) {
#pragma unroll
            for (uint32_t j = k >> 1; j > 0; j >>= 1) {
                const uint64_t o = __shfl_xor_sync(0xffffffffu, v, j);
                const bool keep_min = ((lane & j) == 0) == ((lane & k) == 0);
                v = keep_min ? (v < o ? v : o) : (v < o ? o : v);
            }
        }
        if (i < np) a[i] = v;
    }
    __syncthreads();
    for (uint32_t run = 32; run < np; run <<= 1) {
        for (uint32_t i = threadIdx.x; i < np; i += blockDim.x) {
            const uint64_t v = a[i];
            const uint32_t r = i / run, pos = i - r * run;
            const uint32_t pb = (r ^ 1u) * run;  // partner run
            const bool left = (r & 1u) == 0;
            uint32_t lo = 0, cnt = run;
            while (cnt > 0) {  // partner keys before v: below it (left run) / not above it (right run)
                const uint32_t half = cnt >> 1;
                const uint64_t x = a[pb + lo + half];
                if (left ? x < v : x <= v) {
                    lo += half + 1;
                    cnt -= half + 1;
                } else {
                    cnt = half;
                }
            }
            b[(r & ~1u) * run + pos + lo] = v;
        }
        __syncthreads();
        uint64_t *t = a;
        a = b;
        b = t;
    }
    return a;
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

// The two-queue merge, one thread.  Leaves (sorted keys) and internal nodes
// (created in non-decreasing weight order) are popped smallest first, leaf
// first on ties.  The heads of both queues live in 4-deep register windows
// (L0..L3 = leaves li..li+3, I0..I3 = internal nodes ii..ii+3, ~0 = none):
// a step decides both pops from L0, L1, I0, I1, shifts the windows by the
// pops with selects, and refills positions 2 and 3 with shared-memory loads
// that the NEXT step only reads in its shifts -- the load latency is off the
// dependency chain.  The node created by a step is written to shared memory
// before the refill loads (so they see it) and patched into positions 0/1
// directly.  W = uint32_t when the total count fits (half the compare/add
// work), else uint64_t.
template <typename W>
__device__ __forceinline__ void huffman_merge(const CbScratch &sc, uint32_t n) {
    constexpr W kNone = (W)~(W)0;
    W *wint = reinterpret_cast<W *>(sc.wint);
    auto leaf = [&](uint32_t i) -> W { return i < n ? (W)(sc.key[i] >> 20) : kNone; };
    uint32_t li = 0, ii = 0, ni = 0;
    W L0 = leaf(0), L1 = leaf(1), L2 = leaf(2), L3 = leaf(3);
    W I0 = kNone, I1 = kNone, I2 = kNone, I3 = kNone;
    for (uint32_t k = 0; k + 1 < n; k++) {
        const bool a_leaf = L0 <= I0;  // first pop
        const W cl = a_leaf ? L1 : L0, ci = a_leaf ? I0 : I1;
        const bool b_leaf = cl <= ci;  // second pop
        const W nw = (a_leaf ? L0 : I0) + (b_leaf ? cl : ci);
        const uint32_t id0 = a_leaf ? li : n + ii;
        const uint32_t id1 = b_leaf ? li + (uint32_t)a_leaf : n + ii + (uint32_t)!a_leaf;
        wint[ni] = nw;
        sc.parent[id0] = n + ni;
        sc.parent[id1] = n + ni;
        const uint32_t dl = (uint32_t)a_leaf + (uint32_t)b_leaf, di = 2u - dl;
        li += dl;
        ii += di;
        const W nL0 = dl == 0 ? L0 : (dl == 1 ? L1 : L2);
        const W nL1 = dl == 0 ? L1 : (dl == 1 ? L2 : L3);
        W nI0 = di == 0 ? I0 : (di == 1 ? I1 : I2);
        W nI1 = di == 0 ? I1 : (di == 1 ? I2 : I3);
        if (ni == ii) nI0 = nw;          // the new node is the internal head
        if (ni == ii + 1) nI1 = nw;      // ... or the one after it
        ni++;
        L0 = nL0;
        L1 = nL1;
        L2 = leaf(li + 2);
        L3 = leaf(li + 3);
        I0 = nI0;
        I1 = nI1;
        I2 = ii + 2 < ni ? wint[ii + 2] : kNone;
        I3 = ii + 3 < ni ? wint[ii + 3] : kNone;
    }
}

// The u32 two-queue merge for books in shared memory, one thread, six-deep
// register windows: L0..L5 = leaf weights li..li+5 (lw is padded with the
// "none" marker past n), I0..I5 = internal weights ii..ii+5 (wi starts as
// all "none", so an unwritten slot reads as an empty queue).  A step takes
// both pops from L0/I0 and the first pop's survivors (X0 / Y0), shifts both
// windows with selects, patches the new node into positions 0..3, and
// reloads positions 4 and 5 -- which the next step reads only in its
// selects, a full step after the load, so shared-memory latency never sits
// on the compare -> select -> compare chain.
__device__ __forceinline__ void huffman_merge32(const uint32_t *lw, uint32_t *wi, uint32_t *parent, uint32_t n) {
    uint32_t L0 = lw[0], L1 = lw[1], L2 = lw[2], L3 = lw[3], L4 = lw[4], L5 = lw[5];
    uint32_t I0 = wi[0], I1 = wi[1], I2 = wi[2], I3 = wi[3], I4 = wi[4], I5 = wi[5];
    uint32_t li = 0, ii = 0;
    for (uint32_t ni = 0; ni + 1 < n; ni++) {
        const bool a = L0 <= I0;  // first pop: a leaf (ties go to leaves)
        const uint32_t X0 = a ? L1 : L0, X1 = a ? L2 : L1, X2 = a ? L3 : L2, X3 = a ? L4 : L3, X4 = a ? L5 : L4;
        const uint32_t Y0 = a ? I0 : I1, Y1 = a ? I1 : I2, Y2 = a ? I2 : I3, Y3 = a ? I3 : I4, Y4 = a ? I4 : I5;
        const bool b = X0 <= Y0;  // second pop
        const uint32_t nw = min(L0, I0) + min(X0, Y0);
        const uint32_t pv = n + ni;
        parent[a ? li : n + ii] = pv;
        const uint32_t li1 = li + (uint32_t)a, ii1 = ii + (uint32_t)!a;
        parent[b ? li1 : n + ii1] = pv;
        wi[ni] = nw;
        li = li1 + (uint32_t)b;
        ii = ii1 + (uint32_t)!b;
        L0 = b ? X1 : X0;
        L1 = b ? X2 : X1;
        L2 = b ? X3 : X2;
        L3 = b ? X4 : X3;
        I0 = b ? Y0 : Y1;
        I1 = b ? Y1 : Y2;
        I2 = b ? Y2 : Y3;
        I3 = b ? Y3 : Y4;
        const uint32_t pos = ni - ii;  // the new node's place in the internal window
        I0 = pos == 0 ? nw : I0;
        I1 = pos == 1 ? nw : I1;
        I2 = pos == 2 ? nw : I2;
        I3 = pos == 3 ? nw : I3;
        L4 = lw[li + 4];
        L5 = lw[li + 5];
        I4 = wi[ii + 4];
        I5 = wi[ii + 5];
    }
}

// kSmem: small books, the whole tree lives in shared memory (the pointers
// are derived from the shared array in this instantiation, so the compiler
// emits LDS/STS instead of generic loads -- the serial merge is latency bound)
template <bool kSmem>
__global__ void __launch_bounds__(kCbThreads) k_codebook(const unsigned long long *hist, uint32_t cap,
                                                        uint8_t *lengths, uint64_t *codes,
                                                        lzb_dstatus *st, CbScratch sc, uint32_t npow2) {
    extern __shared__ __align__(16) unsigned char cb_smem[];
    const long long t0 = clock64();  // phase clocks -> st->u[4..5] (diagnostics)
    __shared__ long long s_clk[4];
    if constexpr (kSmem) {
        sc.key = reinterpret_cast<uint64_t *>(cb_smem);
        sc.wint = sc.key + npow2;
        sc.parent = reinterpret_cast<uint32_t *>(sc.wint + cap);
        sc.depth = reinterpret_cast<uint8_t *>(sc.parent + 2 * cap);
    }
    // code lengths: a shared copy for the small-book instantiation (the
    // canonical pass and the stats read them back), copied out once at the end
    uint8_t *len = lengths;
    if constexpr (kSmem)
        len = reinterpret_cast<uint8_t *>(reinterpret_cast<uint32_t *>(sc.depth + 2 * cap + 16 - ((2 * cap) & 15)) +
                                          cap + 16);
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
        if (s < cap) len[s] = 0;
        if (f >= (1ull << 44)) s_err = 1;
        unsigned long long fs = f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) fs += __shfl_xor_sync(0xffffffffu, fs, o);
        if ((threadIdx.x & 31) == 0 && fs) atomicAdd(&s_tot, fs);
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
    {  // keys past n are ~0: sorting the power-of-two prefix covering n suffices
        uint32_t np = 1;
        while (np < n) np <<= 1;
        if (kSmem && np <= cap) {
            // merge sort ping-ponging with wint (cap x u64, unused until the merge)
            uint64_t *sorted = sort_u64_merge(sc.key, sc.wint, np, npow2);
            if (sorted != sc.key) {  // equal-sized arrays: swap the roles
                sc.wint = sc.key;
                sc.key = sorted;
            }
        } else {
            bitonic_sort_u64(sc.key, np);
        }
    }
    if (threadIdx.x == 0) s_clk[0] = clock64() - t0;
    if (n == 1) {
        if (threadIdx.x == 0) len[sc.key[0] & 0xFFFFF] = 1;  // lone symbol -> 1 bit
    } else {
        // two-queue Huffman merge (sequential; n-1 steps) on thread 0; see
        // huffman_merge32 / huffman_merge for the register windows that keep
        // shared-memory latency off the step's dependency chain
        const bool w32 = s_tot < (1ull << 32) - 1;  // every weight below the u32 "none" marker
        if (kSmem && w32 && n + 8 <= 2 * cap) {  // wint holds 2 cap u32 slots
            uint32_t *lw = reinterpret_cast<uint32_t *>(sc.depth + 2 * cap + 16 - ((2 * cap) & 15));
            uint32_t *wi = reinterpret_cast<uint32_t *>(sc.wint);
            for (uint32_t i = threadIdx.x; i < n + 8; i += blockDim.x) {
                lw[i] = i < n ? (uint32_t)(sc.key[i] >> 20) : 0xFFFFFFFFu;
                wi[i] = 0xFFFFFFFFu;
            }
            __syncthreads();
            if (threadIdx.x == 0) huffman_merge32(lw, wi, sc.parent, n);
        } else if (threadIdx.x == 0) {
            if (w32)
                huffman_merge<uint32_t>(sc, n);
            else
                huffman_merge<uint64_t>(sc, n);
        }
        if (threadIdx.x == 0) s_clk[1] = clock64() - t0;
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
            len[sc.key[i] & 0xFFFFF] = (uint8_t)d;
        }
    }
    __syncthreads();
    if (s_err) {
        if (threadIdx.x == 0) set_status(st, LZB_E_DATA);  // code longer than 64 bits
        return;
    }
    if (threadIdx.x == 0) s_clk[2] = clock64() - t0;
    if constexpr (kSmem) {
        for (uint32_t i = threadIdx.x; i < cap; i += blockDim.x) lengths[i] = len[i];
    }
    int rc = canonical_from_lengths(len, cap, codes, s_cnt, s_first, s_misc, false);
    if (rc) {
        if (threadIdx.x == 0) set_status(st, LZB_E_DATA);
        return;
    }
    // exact <b> inputs: sum(count * len) and total
    unsigned long long sum = 0;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {  // the n used symbols, from the sorted keys
        const uint64_t k = sc.key[i];
        sum += (k >> 20) * len[k & 0xFFFFF];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);  // warp sums first
    if ((threadIdx.x & 31) == 0 && sum) atomicAdd(&s_sum, sum);
    __syncthreads();
    if (threadIdx.x == 0) {
        st->u[0] = s_sum;
        st->u[1] = s_tot;
        st->u[2] = s_misc[1];
        st->u[3] = n;
        st->u[4] = (uint64_t)(uint32_t)s_clk[0] | (uint64_t)(uint32_t)s_clk[1] << 32;
        st->u[5] = (uint64_t)(uint32_t)s_clk[2] | (uint64_t)(uint32_t)(clock64() - t0) << 32;
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
    // key | wint | parent | depth | (16-aligned) u32 leaf weights for the merge window | lengths
    size_t smem = (size_t)np * 8 + (size_t)cap * 8 + (size_t)cap * 8 + (size_t)cap * 2 + 16 + ((size_t)cap + 16) * 4 + (size_t)cap;
    int use_smem = smem <= 160 * 1024;
    if (use_smem) {
        LZB_CUDA_TRY(set_dyn_smem(k_codebook<true>, smem));
        k_codebook<true><<<1, kCbThreads, smem, s>>>((const unsigned long long *)hist, cap, lengths, codes,
                                                     st, c, np);
    } else {
        k_codebook<false><<<1, kCbThreads, 0, s>>>((const unsigned long long *)hist, cap, lengths, codes,
                                                   st, c, np);
    }
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
