// K3 Huffman bit packing and K5 self-synchronising parallel Huffman decode.
//
// Reference semantics (P = /root/reference/pkg/src/lzebc):
//   encode            P/huffman.py:46-61   MSB-first concatenation of code words,
//                                          last byte zero padded, NO per-chunk
//                                          offsets anywhere (dense stream)
//   _decode_tables    P/huffman.py:64-82   canonical first/limit/offset tables
//   _decode_kernel    P/huffman.py:85-106  bit-serial; -1 code > 64 bits,
//                                          -2 too many code words, -3 stream ends
//                                          mid code word
//   decode            P/huffman.py:109-122 count mismatch -> CorruptArchiveError
//
// K3: tiles of 4096 symbols; per-thread bit counts -> block scan ->
// decoupled look-back gives the tile's u64 bit offset in ONE pass over the
// symbols.  Code words are OR-ed into a shared-memory word buffer; words fully
// inside the tile are stored directly (big-endian byte order), the <= 2 partial
// boundary words per tile go through a tiny fix-up pass.
//
// K5: the stream is cut into subsequences of S bits.  For every
// possible entry phase p in [0, maxlen) a thread decodes its subsequence and
// records a transfer map p -> (exit phase, code words started); phases merge
// as soon as they hit a code-word boundary of an already decoded path, so the
// common case costs ~one decode.  A hierarchical composition of the maps gives
// every subsequence's true entry phase and symbol offset with bounded work
// even for non-synchronising (e.g. fixed-length) code books.  A final pass
// decodes from the true entries, staging 32 symbols per lane in shared memory
// so each warp writes coalesced runs.
#include "lzb_common.cuh"
#include "lzb_dectab.cuh"
#define LZB_DEC4_KERNELS
#include "lzb_dec4.cuh"

namespace lzb {

// ============================================================================
// K3 encode
// ============================================================================
constexpr int kEThreads = 256;
constexpr int kESyms = 16;
constexpr int kETile = kEThreads * kESyms;

struct EncParams {
    const void *sym;
    uint64_t n;
    const uint8_t *lengths;
    const uint64_t *codes;
    uint32_t cap;
    uint8_t *out;
    uint64_t out_bytes;
    uint64_t bit_offset;  // phase of the first bit inside out[0] (0..7)
    lzb_dstatus *st;
    uint64_t *lb;
    unsigned int *ticket;
    uint64_t ntiles;
    uint64_t *frag;  // per tile: [head word, head bits, tail word, tail bits] (word = ~0 none)
    uint32_t maxlen;
    int table_smem;
};

__device__ __forceinline__ void store_word_bytes(uint8_t *out, uint64_t byte0, uint32_t be_word,
                                                 uint64_t limit) {
#pragma unroll
    for (int k = 0; k < 4; k++)
        if (byte0 + k < limit) out[byte0 + k] = (uint8_t)(be_word >> (24 - 8 * k));
}

// K3 kernel.  SHORT = every code word has <= 32 bits (the host passes the
// book's max length; practically always true): the table is one u64 per
// symbol (code | len << 32) and each code word is placed branch-free with one
// or two shared-memory ORs.  !SHORT handles 33..64-bit code words generically.
template <typename SymT, bool SHORT, bool TSMEM>
__global__ void __launch_bounds__(kEThreads) k_huff_encode(EncParams p) {
    extern __shared__ __align__(16) unsigned char e_smem[];
    // [table: cap x u64 (code | len << 32) or cap x (u64 code + u8 len)][words]
    uint64_t *s_tab = reinterpret_cast<uint64_t *>(e_smem);
    uint8_t *s_lens = reinterpret_cast<uint8_t *>(s_tab + p.cap);
    const size_t tbytes = TSMEM ? (size_t)p.cap * 9 : 0;
    uint32_t *s_words = reinterpret_cast<uint32_t *>(e_smem + ((tbytes + 15) & ~(size_t)15));
    __shared__ uint32_t s_scan[33];
    __shared__ uint64_t s_tile, s_excl;
    if (TSMEM) {
        for (uint32_t i = threadIdx.x; i < p.cap; i += blockDim.x) {
            if (SHORT) {  // left-aligned 32-bit code word | length << 32
                const uint32_t L = p.lengths[i];
                const uint32_t cal = L ? (uint32_t)(p.codes[i] << (32 - L)) : 0u;
                s_tab[i] = (uint64_t)cal | ((uint64_t)L << 32);
            }
            else {
                s_tab[i] = p.codes[i];
                s_lens[i] = p.lengths[i];
            }
        }
    }
    const uint64_t *tab = TSMEM ? s_tab : p.codes;
    const uint8_t *lens = TSMEM ? s_lens : p.lengths;
    const uint32_t tid = threadIdx.x;
    const uint32_t capm1 = p.cap - 1;
    uint32_t bad = 0;
    while (true) {
        if (tid == 0) s_tile = atomicAdd(p.ticket, 1u);
        __syncthreads();
        const uint64_t t = s_tile;
        if (t >= p.ntiles) break;
        const uint64_t base = t * kETile + (uint64_t)tid * kESyms;
        uint32_t sy[kESyms];
        const SymT *sp = static_cast<const SymT *>(p.sym) + base;
        const bool fullv = base + kESyms <= p.n && sizeof(SymT) == 2 &&
                           (reinterpret_cast<uintptr_t>(sp) & 15) == 0;
        uint32_t nvalid = kESyms;
        if (fullv) {
            uint4 a = reinterpret_cast<const uint4 *>(sp)[0];
            uint4 b = reinterpret_cast<const uint4 *>(sp)[1];
            uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
            for (int k = 0; k < 8; k++) {
                sy[2 * k] = w[k] & 0xFFFFu;
                sy[2 * k + 1] = w[k] >> 16;
            }
        } else {
            nvalid = base >= p.n ? 0u : (uint32_t)umin64(kESyms, p.n - base);
#pragma unroll
            for (int k = 0; k < kESyms; k++) sy[k] = (uint32_t)k < nvalid ? (uint32_t)sp[k] : 0u;
        }
        uint32_t Ls[kESyms];
        uint64_t Cs[kESyms];
        uint32_t nb = 0;
        if (fullv) nvalid = kESyms;
#pragma unroll
        for (int k = 0; k < kESyms; k++) {
            const uint32_t sv = sy[k];
            const uint32_t idx = sv < capm1 ? sv : capm1;
            uint32_t L;
            uint64_t c;
            if (SHORT) {
                if (TSMEM) {
                    const uint64_t e = tab[idx];
                    L = (uint32_t)(e >> 32);
                    c = (uint32_t)e;
                } else {  // big books: raw tables in global memory
                    L = lens[idx];
                    c = L ? (uint32_t)(tab[idx] << (32 - L)) : 0u;
                }
            } else {
                L = lens[idx];
                c = tab[idx];
            }
            const bool v = (uint32_t)k < nvalid;
            bad |= (uint32_t)(v && (sv > capm1 || L == 0));
            L = v ? L : 0u;
            Ls[k] = L;
            Cs[k] = L ? c : 0ull;  // zero-length entries contribute nothing
            nb += L;
        }
        uint32_t tile_bits;
        const uint32_t off = block_exclusive_scan<uint32_t>(nb, s_scan, &tile_bits);
        // publish the aggregate now; resolve after the packing work
        if (tid == 0) lb_store(&p.lb[t], (t == 0 ? kLbInc : kLbAgg) | tile_bits);
        const uint32_t nwords = (tile_bits + 31) >> 5;
        for (uint32_t i = tid; i <= nwords + 1; i += kEThreads) s_words[i] = 0;
        __syncthreads();
        // pack at tile-relative bit offsets (phase 0)
        uint32_t pos = off;
        const uint32_t wbase_s = (uint32_t)__cvta_generic_to_shared(s_words);
#pragma unroll
        for (int k = 0; k < kESyms; k++) {
            const uint32_t L = Ls[k];
            if (SHORT) {
                // code word -> bits [sh, sh + L) of a 64-bit window at word w:
                // two unconditional shared-memory ORs (the second ORs zero
                // unless the code word crosses a word boundary), no branches
                const uint32_t sh = pos & 31;
                const uint32_t addr = wbase_s + ((pos >> 5) << 2);
                const uint64_t v = (Cs[k] << 32) >> sh;  // Cs = left-aligned code word
                asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(addr), "r"((uint32_t)(v >> 32)) : "memory");
                asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(addr + 4), "r"((uint32_t)v) : "memory");
            } else {
                uint32_t rem = L, q = pos;
                const uint64_t c = Cs[k];
                while (rem) {
                    const uint32_t sh = q & 31, take = (32 - sh) < rem ? (32 - sh) : rem;
                    const uint32_t piece = (uint32_t)((c >> (rem - take)) & ((1ull << take) - 1ull));
                    atomicOr(&s_words[q >> 5], piece << (32 - sh - take));
                    rem -= take;
                    q += take;
                }
            }
            pos += L;
        }
        if ((tid >> 5) == 0) {
            uint64_t ex = lb_resolve(p.lb, t, tile_bits);
            if (lane_id() == 0) s_excl = ex;
        }
        __syncthreads();
        // write out with the tile's bit phase: out word j = (w[j-1] << (32-s)) | (w[j] >> s)
        const uint64_t G = s_excl + p.bit_offset;
        const uint32_t sft = (uint32_t)(G & 31);
        const uint64_t wbase = G >> 5;
        const uint64_t endbit = G + tile_bits;
        const uint32_t nout = (uint32_t)(((endbit + 31) >> 5) - wbase);
        const bool aligned = (reinterpret_cast<uintptr_t>(p.out) & 3) == 0;
        for (uint32_t j = tid; j < nout; j += kEThreads) {
            const uint32_t cur = j < nwords ? s_words[j] : 0u;
            const uint32_t prv = j > 0 ? s_words[j - 1] : 0u;
            const uint32_t v = sft ? ((prv << (32 - sft)) | (cur >> sft)) : cur;
            const uint64_t gw = wbase + j;
            const bool full = (gw * 32 >= G) && (gw * 32 + 32 <= endbit);
            if (full) {
                if (aligned) reinterpret_cast<uint32_t *>(p.out)[gw] = bswap32(v);
                else store_word_bytes(p.out, gw * 4, v, ~0ull);
            } else if (j == 0 || j == nout - 1) {
                // partial boundary words go to the fix-up pass
                const bool head = (j == 0) && (sft != 0);
                if (head) {
                    p.frag[4 * t + 0] = gw;
                    p.frag[4 * t + 1] = v;
                }
                if (j == nout - 1 && !(head && nout == 1)) {
                    p.frag[4 * t + 2] = gw;
                    p.frag[4 * t + 3] = v;
                }
            }
        }
        if (tid == 0) {
            const bool has_head = tile_bits > 0 && sft != 0;
            const bool has_tail = tile_bits > 0 && (endbit & 31) != 0 && !(has_head && nout == 1);
            if (!has_head) p.frag[4 * t + 0] = ~0ull;
            if (!has_tail) p.frag[4 * t + 2] = ~0ull;
            if (t == p.ntiles - 1) p.st->u[0] = s_excl + tile_bits;
        }
        __syncthreads();
    }
    if (__any_sync(0xffffffffu, bad != 0) && lane_id() == 0) set_status(p.st, LZB_E_DATA);
}

// Boundary words: each partial word is shared by at most the tail of tile t
// and the head of tile t+1 (every tile but the last spans >= 4096 bits).
__global__ void k_huff_fixup(EncParams p) {
    const uint64_t nbytes = umin64(p.out_bytes, (p.bit_offset + p.st->u[0] + 7) / 8);
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < p.ntiles;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t hw = p.frag[4 * t], hb = p.frag[4 * t + 1];
        const uint64_t tw = p.frag[4 * t + 2], tb = p.frag[4 * t + 3];
        if (hw != ~0ull) {
            uint32_t v = (uint32_t)hb;
            if (t > 0) {
                if (p.frag[4 * (t - 1) + 2] == hw) v |= (uint32_t)p.frag[4 * (t - 1) + 3];
                else if (p.frag[4 * (t - 1)] == hw) v |= (uint32_t)p.frag[4 * (t - 1) + 1];
            }
            store_word_bytes(p.out, hw * 4, v, nbytes);
        }
        if (tw != ~0ull) {
            bool shared = t + 1 < p.ntiles && p.frag[4 * (t + 1)] == tw;
            if (!shared) store_word_bytes(p.out, tw * 4, (uint32_t)tb, nbytes);
        }
    }
}

// ----------------------------------------------------------------------------
// K3 fast path (u16 symbols, code words <= 32 bits, table in shared memory).
// A warp tile is 1024 symbols; lane l owns the 32 consecutive symbols
// [32 l, 32 l + 32), i.e. the four 16-byte pieces 4l..4l+3.  Three kernels:
//   k_huff_count_w: bit count of every tile and of every lane's 32 symbols
//                   (order-independent coalesced loads; the DataError checks);
//   k_huff_scan_w:  single-pass look-back scan -> u64 bit offset per tile;
//   k_huff_encode_w: persistent warps (tile t to warp t mod NW, 4 CTAs/SM),
//                   the next tile prefetched by cp.async into the warp's one
//                   XOR-swizzled stage as soon as the lanes hold the current
//                   one in registers; each lane packs its code words into a
//                   32-bit accumulator and stores every word it completes
//                   (its partial first / last word via red.shared.or), then
//                   the warp stores the tile's words big-endian with the
//                   tile's bit phase applied and keeps the <= 2 partial
//                   boundary words (head / tail) for k_huff_fixup_w.
// ----------------------------------------------------------------------------
constexpr int kWSyms = 32;                 // symbols per lane
constexpr int kWTile = 32 * kWSyms;        // 1024 symbols per warp tile
constexpr int kWWarps = 8;

__device__ __forceinline__ uint32_t sym16(const uint4 &v, int k) {
    const uint32_t w = k < 2 ? v.x : k < 4 ? v.y : k < 6 ? v.z : v.w;
    return (k & 1) ? (w >> 16) : (w & 0xFFFFu);
}

struct EncWParams {
    const uint16_t *sym;
    uint64_t n;
    const uint8_t *lengths;
    const uint64_t *codes;
    uint32_t cap;
    uint8_t *out;
    uint64_t bit_offset;
    lzb_dstatus *st;
    uint32_t *cnt;         // per warp tile bit count (+1 zero entry)
    uint16_t *lcnt;        // per warp tile x lane: bits of the lane's 32 symbols
    uint64_t *toff;        // exclusive scan of cnt: tile bit offsets, toff[ntiles] = total
    uint64_t *lb;          // scan look-back words
    unsigned int *ticket;  // scan ticket
    uint32_t *frag;        // per warp tile: [head partial word, tail partial word]
    uint64_t ntiles;
    uint32_t wwords;       // per-warp word buffer (u32)
};

// Pass A: bit count of every warp tile (order-independent, so lane l simply
// takes the 16-byte pieces l, l+32, l+64, l+96: coalesced 16-byte loads).
// Also the DataError checks (symbol >= cap, symbol without a code word).
__global__ void __launch_bounds__(256) k_huff_count_w(const __grid_constant__ EncWParams p) {
    __shared__ uint8_t s_len[4096];
    // code words over 32 bits (possible only when the book was built on the
    // device in this stream, LZB_MAXLEN_DEVICE): counted as 32 so every
    // offset stays inside the buffers sized for 32, and reported as RETRY
    int longer = 0;
    for (uint32_t i = threadIdx.x; i < p.cap; i += blockDim.x) {
        const uint32_t L = p.lengths[i];
        longer |= L > 32;
        s_len[i] = (uint8_t)(L > 32 ? 32 : L);
    }
    if (__syncthreads_or(longer)) {
        if (threadIdx.x == 0) set_status(p.st, LZB_E_RETRY);
    }
    const uint32_t lane = lane_id();
    const uint64_t NW = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t capm1 = p.cap - 1;
    const bool aligned_in = (reinterpret_cast<uintptr_t>(p.sym) & 15) == 0;
    uint32_t mx = 0, mnL = 64;
    for (uint64_t t = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; t < p.ntiles; t += NW) {
        const bool full = aligned_in && (t + 1) * kWTile <= p.n;
        uint32_t pc[4] = {0, 0, 0, 0};  // bits of pieces lane, lane+32, lane+64, lane+96
        if (full) {
            const uint4 *src = reinterpret_cast<const uint4 *>(p.sym + t * kWTile);
            uint4 v[4];
#pragma unroll
            for (int j = 0; j < 4; j++) v[j] = __ldcs(src + j * 32 + lane);
#pragma unroll
            for (int i = 0; i < 32; i++) {
                const uint32_t sv = sym16(v[i >> 3], i & 7);
                const uint32_t L = s_len[sv < capm1 ? sv : capm1];
                mx = sv > mx ? sv : mx;
                mnL = L < mnL ? L : mnL;
                pc[i >> 3] += L;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 4; j++) {
                for (uint32_t k = 0; k < 8; k++) {
                    const uint64_t g = t * kWTile + (uint64_t)(j * 32 + lane) * 8 + k;
                    if (g >= p.n) break;
                    const uint32_t sv = p.sym[g];
                    const uint32_t L = s_len[sv < capm1 ? sv : capm1];
                    mx = sv > mx ? sv : mx;
                    mnL = L < mnL ? L : mnL;
                    pc[j] += L;
                }
            }
        }
        // encode lane l owns pieces 4l..4l+3: piece q sits in lane q & 31, slot q >> 5 = l >> 3
        const uint32_t p01 = pc[0] | (pc[1] << 16), p23 = pc[2] | (pc[3] << 16);
        uint32_t mine = 0;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const uint32_t src = 4 * (lane & 7) + k;
            const uint32_t a01 = __shfl_sync(0xffffffffu, p01, src);
            const uint32_t a23 = __shfl_sync(0xffffffffu, p23, src);
            const uint32_t sel = lane >> 3;
            const uint32_t w = sel < 2 ? a01 : a23;
            mine += (sel & 1) ? (w >> 16) : (w & 0xFFFFu);
        }
        p.lcnt[t * 32 + lane] = (uint16_t)mine;
        const uint32_t nb = __reduce_add_sync(0xffffffffu, mine);
        if (lane == 0) p.cnt[t] = nb;
    }
    const bool bad = mx > capm1 || mnL == 0;
    if (__any_sync(0xffffffffu, bad) && lane == 0) set_status(p.st, LZB_E_DATA);
}

// exclusive scan of the ntiles + 1 tile counts -> u64 bit offsets
__global__ void __launch_bounds__(256) k_huff_scan_w(const __grid_constant__ EncWParams p) {
    __shared__ uint64_t s_t, s_ex;
    __shared__ uint64_t s_scan[33];
    const uint64_t n = p.ntiles + 1;
    if (threadIdx.x == 0) s_t = atomicAdd(p.ticket, 1u);
    __syncthreads();
    const uint64_t t = s_t;
    const uint64_t base = t * 2048 + (uint64_t)threadIdx.x * 8;
    uint64_t v[8], sum = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        v[k] = base + k < n ? p.cnt[base + k] : 0;
        sum += v[k];
    }
    uint64_t total;
    const uint64_t off = block_exclusive_scan<uint64_t>(sum, s_scan, &total);
    if ((threadIdx.x >> 5) == 0) {
        const uint64_t ex = lookback_warp(p.lb, t, total);
        if (lane_id() == 0) s_ex = ex;
    }
    __syncthreads();
    uint64_t run = s_ex + off;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        if (base + k < n) p.toff[base + k] = run;
        run += v[k];
    }
}

// stage slot of 16-byte piece q (0..127): conflict-free for lane l reading 4l+k
__device__ __forceinline__ uint32_t wswz(uint32_t q) { return q ^ ((q >> 3) & 7u); }

// Pack one lane's 32 code words at tile-relative bit `off` with a 32-bit
// accumulator, four (or two) symbols per step when their code words fit 32
// bits together.  Every word the lane COMPLETES is stored plainly (only the lane
// holding a word's last bit completes it; bits of earlier lanes in that word
// are zero here and are OR-ed in afterwards); the lane's final partial word is
// returned for a red.shared.or after a __syncwarp.
template <bool FULL>
__device__ __forceinline__ void enc_pack_lane(const uint4 (&v)[4], uint32_t nv, uint32_t off,
                                              uint32_t words_s, const uint64_t *s_tab,
                                              uint32_t capm1, uint32_t &last_addr,
                                              uint32_t &last_val, uint32_t &last_n) {
    uint32_t n = off & 31, cur = 0;
    uint32_t waddr = words_s + ((off >> 5) << 2);
    // one accumulator step for a left-aligned code word c of L <= 32 bits
    auto step = [&](uint32_t c, uint32_t L) {
        cur |= c >> n;
        const uint32_t nn = n + L;
        const uint32_t f = nn >= 32 ? 1u : 0u;
        asm volatile("{\n\t.reg .pred ps;\n\tsetp.ne.u32 ps, %2, 0;\n\t@ps st.shared.u32 [%0], %1;\n\t}"
                     ::"r"(waddr), "r"(cur), "r"(f)
                     : "memory");
        const uint32_t rem = __funnelshift_lc(0u, c, 32 - n);  // bits that did not fit
        cur = f ? rem : cur;
        waddr += f << 2;
        n = nn - (f << 5);
    };
    // symbols in quads: four code words that fit 32 bits together take one
    // step; otherwise pairs, otherwise single code words.  (cap is a power of
    // two: masking keeps an invalid symbol's lookup in range; the count pass
    // has already flagged it as a DataError.)
#pragma unroll
    for (int i = 0; i < kWSyms / 4; i++) {
        const uint4 &q = v[i >> 1];
        const uint32_t wa = (i & 1) ? q.z : q.x, wb = (i & 1) ? q.w : q.y;
        const uint64_t e0 = s_tab[wa & capm1], e1 = s_tab[(wa >> 16) & capm1];
        const uint64_t e2 = s_tab[wb & capm1], e3 = s_tab[(wb >> 16) & capm1];
        uint32_t L0 = (uint32_t)(e0 >> 32), L1 = (uint32_t)(e1 >> 32);
        uint32_t L2 = (uint32_t)(e2 >> 32), L3 = (uint32_t)(e3 >> 32);
        uint32_t c0 = (uint32_t)e0, c1 = (uint32_t)e1, c2 = (uint32_t)e2, c3 = (uint32_t)e3;
        if (!FULL) {
            const uint32_t b = 4 * i;
            L0 = b < nv ? L0 : 0u;
            c0 = L0 ? c0 : 0u;
            L1 = b + 1 < nv ? L1 : 0u;
            c1 = L1 ? c1 : 0u;
            L2 = b + 2 < nv ? L2 : 0u;
            c2 = L2 ? c2 : 0u;
            L3 = b + 3 < nv ? L3 : 0u;
            c3 = L3 ? c3 : 0u;
        }
        const uint32_t La = L0 + L1, Lb = L2 + L3;
        if (La + Lb <= 32) {
            const uint32_t ca = c0 | __funnelshift_rc(c1, 0u, L0);  // c1 >> L0 (0 for L0 == 32)
            const uint32_t cb = c2 | __funnelshift_rc(c3, 0u, L2);
            step(ca | __funnelshift_rc(cb, 0u, La), La + Lb);
        } else {
            if (La <= 32) {
                step(c0 | __funnelshift_rc(c1, 0u, L0), La);
            } else {
                step(c0, L0);
                step(c1, L1);
            }
            if (Lb <= 32) {
                step(c2 | __funnelshift_rc(c3, 0u, L2), Lb);
            } else {
                step(c2, L2);
                step(c3, L3);
            }
        }
    }
    last_addr = waddr;
    last_val = cur;
    last_n = n;
}

__global__ void __launch_bounds__(kWWarps * 32, 4) k_huff_encode_w(const __grid_constant__ EncWParams p) {
    extern __shared__ __align__(16) unsigned char ew_smem[];
    // [table: cap x u64 (left-aligned code | len << 32)][stage: warps x 2 KB]
    // [words: warps x wwords u32]
    uint64_t *s_tab = reinterpret_cast<uint64_t *>(ew_smem);
    unsigned char *stage_all = ew_smem + (((size_t)p.cap * 8 + 15) & ~(size_t)15);
    uint32_t *words_all = reinterpret_cast<uint32_t *>(stage_all + kWWarps * kWTile * 2);
    for (uint32_t i = threadIdx.x; i < p.cap; i += blockDim.x) {
        const uint32_t L = p.lengths[i];
        const uint32_t cal = (L && L <= 32) ? (uint32_t)(p.codes[i] << (32 - L)) : 0u;
        s_tab[i] = (uint64_t)cal | ((uint64_t)(L > 32 ? 32 : L) << 32);  // > 32: RETRY (count pass)
    }
    __syncthreads();
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    const uint64_t NW = (uint64_t)gridDim.x * kWWarps;
    uint64_t t = (uint64_t)blockIdx.x * kWWarps + warp;
    unsigned char *stage = stage_all + warp * kWTile * 2;
    const uint32_t stage_s = (uint32_t)__cvta_generic_to_shared(stage);
    uint32_t *words = words_all + warp * p.wwords;
    const uint32_t words_s = (uint32_t)__cvta_generic_to_shared(words);
    const uint32_t capm1 = p.cap - 1;
    const bool aligned_out = (reinterpret_cast<uintptr_t>(p.out) & 3) == 0;
    const bool aligned_in = (reinterpret_cast<uintptr_t>(p.sym) & 15) == 0;

    auto is_full = [&](uint64_t tt) { return aligned_in && (tt + 1) * kWTile <= p.n; };
    auto prefetch = [&](uint64_t tt) {
        const unsigned char *src = reinterpret_cast<const unsigned char *>(p.sym + tt * kWTile);
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const uint32_t q = j * 32 + lane;  // coalesced global pieces
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(stage_s + wswz(q) * 16),
                         "l"(src + q * 16)
                         : "memory");
        }
    };
    if (t < p.ntiles && is_full(t)) prefetch(t);
    asm volatile("cp.async.commit_group;" ::: "memory");
    // the lane count and tile offset are loaded one tile ahead (latency)
    uint32_t nb_nx = t < p.ntiles ? p.lcnt[t * 32 + lane] : 0u;
    uint64_t ex_nx = t < p.ntiles ? p.toff[t] : 0ull;
    for (; t < p.ntiles; t += NW) {
        const uint64_t tn = t + NW;
        const uint32_t nb = nb_nx;
        const uint64_t ex = ex_nx;
        if (tn < p.ntiles) {
            nb_nx = p.lcnt[tn * 32 + lane];
            ex_nx = p.toff[tn];
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();  // lanes read pieces other lanes copied
        const bool full = is_full(t);
        const uint64_t b0 = t * kWTile + (uint64_t)lane * kWSyms;
        // ---- the lane's 32 symbols (into registers; the stage is then free) ----
        uint4 v[4];
        uint32_t nv = kWSyms;
        if (full) {
#pragma unroll
            for (int k = 0; k < 4; k++)
                v[k] = *reinterpret_cast<const uint4 *>(stage + wswz(4 * lane + k) * 16);
        } else {
            nv = b0 >= p.n ? 0u : (uint32_t)umin64(kWSyms, p.n - b0);
#pragma unroll
            for (int k = 0; k < 4; k++) {
                uint32_t w[4];
#pragma unroll
                for (int h = 0; h < 4; h++) {
                    const uint32_t i0 = 8 * k + 2 * h;
                    const uint32_t lo = i0 < nv ? (uint32_t)p.sym[b0 + i0] : 0u;
                    const uint32_t hi = i0 + 1 < nv ? (uint32_t)p.sym[b0 + i0 + 1] : 0u;
                    w[h] = lo | (hi << 16);
                }
                v[k] = make_uint4(w[0], w[1], w[2], w[3]);
            }
        }
        __syncwarp();  // every lane holds its pieces: refill the stage with the next tile
        if (tn < p.ntiles && is_full(tn)) prefetch(tn);
        asm volatile("cp.async.commit_group;" ::: "memory");
        // ---- lane bit offsets from the count pass ----
        uint32_t inc = nb;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t a = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= (uint32_t)o) inc += a;
        }
        const uint32_t tile_bits = __shfl_sync(0xffffffffu, inc, 31);
        const uint32_t off = inc - nb;
        const uint32_t nwords = (tile_bits + 31) >> 5;
        for (uint32_t i = lane; i <= nwords; i += 32) words[i] = 0;
        __syncwarp();
        // ---- pass 2: accumulate, store completed words (branch-free) ----
        uint32_t la, lv, ln;
        if (full) enc_pack_lane<true>(v, kWSyms, off, words_s, s_tab, capm1, la, lv, ln);
        else enc_pack_lane<false>(v, nv, off, words_s, s_tab, capm1, la, lv, ln);
        __syncwarp();
        if (ln) asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(la), "r"(lv) : "memory");
        __syncwarp();
        // ---- store with the tile's bit phase ----
        const uint64_t G = ex + p.bit_offset;
        const uint32_t sft = (uint32_t)(G & 31);
        const uint64_t wbase = G >> 5;
        const uint64_t endbit = G + tile_bits;
        const uint32_t nout = tile_bits ? (uint32_t)(((endbit + 31) >> 5) - wbase) : 0u;
        for (uint32_t jw = lane; jw < nout; jw += 32) {
            const uint32_t cw = jw < nwords ? words[jw] : 0u;
            const uint32_t pw = jw > 0 ? words[jw - 1] : 0u;
            const uint32_t val = sft ? ((pw << (32 - sft)) | (cw >> sft)) : cw;
            const uint64_t gw = wbase + jw;
            const bool head = jw == 0 && sft != 0;
            const bool tail = jw == nout - 1 && (endbit & 31) != 0;
            if (!head && !tail) {
                if (aligned_out) reinterpret_cast<uint32_t *>(p.out)[gw] = bswap32(val);
                else store_word_bytes(p.out, gw * 4, val, ~0ull);
            } else {
                // a single-word tile keeps its one partial word as the head
                if (head) p.frag[2 * t] = val;
                else p.frag[2 * t + 1] = val;
            }
        }
        __syncwarp();
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
}

// Partial boundary words of the warp tiles.  Tile t covers global bits
// [G_t, E_t) (inclusive look-back prefixes + bit_offset).  A partial head
// word of t (G_t % 32 != 0) is shared with the partial tail of t-1 (every
// tile but the last spans > 32 bits), so the head owner writes both; a
// partial tail is written by its own tile only when no tile follows.
__global__ void k_huff_fixup_w(const __grid_constant__ EncWParams p) {
    const uint64_t total = p.bit_offset + p.toff[p.ntiles];
    const uint64_t nbytes = (total + 7) / 8;
    if (blockIdx.x == 0 && threadIdx.x == 0) p.st->u[0] = p.toff[p.ntiles];
    const bool aligned = (reinterpret_cast<uintptr_t>(p.out) & 3) == 0;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < p.ntiles;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t G = p.bit_offset + p.toff[t];
        const uint64_t E = p.bit_offset + p.toff[t + 1];
        if (E == G) continue;
        const uint64_t hw = G >> 5, tw = (E - 1) >> 5;
        const bool head = (G & 31) != 0;
        const bool tail = (E & 31) != 0 && !(head && tw == hw);
        if (head) {
            uint32_t v = p.frag[2 * t];
            if (t > 0) {  // the previous tile's partial tail (or its single-word head)
                const uint64_t Gp = p.bit_offset + p.toff[t - 1];
                const bool prev_single = (Gp & 31) != 0 && (Gp >> 5) == hw;
                v |= prev_single ? p.frag[2 * (t - 1)] : p.frag[2 * (t - 1) + 1];
            }
            if (aligned && hw * 4 + 4 <= nbytes) reinterpret_cast<uint32_t *>(p.out)[hw] = bswap32(v);
            else store_word_bytes(p.out, hw * 4, v, nbytes);
        }
        if (tail && t + 1 == p.ntiles) store_word_bytes(p.out, tw * 4, p.frag[2 * t + 1], nbytes);
    }
}

// ============================================================================
// K5 decode
// ============================================================================
struct DecParams {
    const uint32_t *words;  // 4-byte aligned base covering the stream
    uint32_t head;          // bit offset of the stream inside words[0]
    uint64_t nwords;
    uint64_t bit_len;
    uint64_t count;
    const DecTables *tab;
    const uint32_t *syms;  // symbols sorted by (length, symbol)
    uint32_t S;            // subsequence length in bits (multiple of 32)
    uint64_t T;            // subsequences
    uint32_t P;            // phases per subsequence (= maxlen)
    uint32_t *maps;        // T * P entries: (count << 8) | exit
    lzb_dstatus *st;
    void *out;
    // resolution
    uint32_t G;        // group size
    uint64_t ng1, ng2;
    uint64_t *g1;      // ng1 * P : (count << 8) | exit
    uint64_t *g2;      // ng2 * P
    uint8_t *ent2;     // per level-2 group: entry phase
    uint64_t *off2;    // per level-2 group: symbol offset
    uint8_t *ent1;
    uint64_t *off1;
    uint8_t *ent0;     // per subsequence
    uint64_t *off0;
    uint16_t *cp;      // v3: per microblock (count << 8) | chain entry offset
    uint64_t *irr;     // v3: per subsequence, entry phases that join the chain late
    uint8_t *uexit;    // per subsequence: the exit shared by all valid entry phases (0xFF: none)
    unsigned int *nonuni;  // count of subsequences whose valid entries exit differently
    uint64_t *ulb;     // look-back words of the uniform scan
    unsigned int *uticket;
    // plan mode (K5 v4, lzb_dec4.cuh): entries from the plan's per-microblock
    // cp (above), offsets per subsequence, no irregular entries
    const uint64_t *psoff;
    const uint8_t *pirr;
    // bit-range mode (multi-GPU decode of one stream, lzb_huff_range_*):
    // the range starts in phase entry0 and must leave in phase exit_expect
    // (kExitEnd when it ends the stream); an open range's last subsequence
    // is an ordinary one, and code words may run past bit_len up to total_bits.
    uint32_t entry0, exit_expect, open_end;
    uint64_t total_bits;
};

__device__ __forceinline__ uint32_t bswap_load(const DecParams &p, uint64_t w) {
    return w < p.nwords ? bswap32(__ldg(&p.words[w])) : 0u;
}

// 64 bits starting at absolute stream bit q (MSB aligned)
__device__ __forceinline__ uint64_t peek64(const DecParams &p, uint64_t q) {
    uint64_t a = q + p.head;
    uint64_t w = a >> 5;
    uint32_t b = a & 31;
    uint64_t hi = ((uint64_t)bswap_load(p, w) << 32) | bswap_load(p, w + 1);
    if (b == 0) return hi;
    uint64_t nx = bswap_load(p, w + 2);
    return (hi << b) | (nx >> (32 - b));
}

__device__ __forceinline__ uint32_t lm_count(uint64_t e) { return (uint32_t)(e & 3u); }
__device__ __forceinline__ uint32_t lm_len(uint64_t e, int i) { return (uint32_t)(e >> (2 + 4 * i)) & 15u; }
__device__ __forceinline__ uint32_t lm_sym(uint64_t e, int i) { return (uint32_t)(e >> (16 + 16 * i)) & 0xFFFFu; }

// Branch-free bit window for the decode loops: two consecutive stream words
// (w0:w1) and the bit offset sh < 32 of the current position inside w0.
// peek12() = next 12 bits; consume(L <= 32) advances, pulling the next word
// (predicated load, L1-resident stream) when the position leaves w0.
struct Win {
    uint64_t wi;  // word index of w0
    uint32_t w0, w1, w2, w3, sh;  // w2/w3 are prefetched: a load is needed ~3 words later
    __device__ __forceinline__ void init(const DecParams &p, uint64_t q) {
        const uint64_t a = q + p.head;
        wi = a >> 5;
        sh = (uint32_t)(a & 31);
        w0 = bswap_load(p, wi);
        w1 = bswap_load(p, wi + 1);
        w2 = bswap_load(p, wi + 2);
        w3 = bswap_load(p, wi + 3);
    }
    __device__ __forceinline__ uint32_t peek32() const { return __funnelshift_l(w1, w0, sh); }
    __device__ __forceinline__ uint32_t peek12() const { return peek32() >> (32 - kLutBits); }
    __device__ __forceinline__ void consume(const DecParams &p, uint32_t L) {
        sh += L;
        if (sh >= 32) {
            sh -= 32;
            wi++;
            w0 = w1;
            w1 = w2;
            w2 = w3;
            w3 = bswap_load(p, wi + 3);
        }
    }
    __device__ __forceinline__ uint64_t abs_pos(const DecParams &p) const { return wi * 32 + sh - p.head; }
};

// Long code word (> 12 bits) or invalid prefix at absolute bit q: canonical
// tables on 64 peeked bits.  Returns len (0 = invalid), *sym.
__device__ __forceinline__ uint32_t decode_long(const DecParams &p, const DecCanon *tab, uint64_t q,
                                                uint32_t &sym) {
    const uint64_t v = peek64(p, q);
    // from length 1: books with cap > 65536 have no symbols in the LUTs
    for (uint32_t L = 1; L <= tab->maxlen; L++) {
        const uint64_t c = v >> (64 - L);
        const uint64_t f = tab->first[L], k = tab->cnt[L];
        if (k && c >= f && c - f < k) {
            sym = p.syms[tab->off[L] + (uint32_t)(c - f)];
            return L;
        }
    }
    return 0;
}

__global__ void k_dec_tables(const uint8_t *lengths, uint32_t cap, uint32_t maxlen_hint,
                             DecTables *tab, uint32_t *syms, lzb_dstatus *st) {
    __shared__ uint32_t s_cnt[65];
    __shared__ uint32_t s_off[65];
    __shared__ uint32_t s_bad, s_max;
    for (uint32_t i = threadIdx.x; i < 65; i += blockDim.x) s_cnt[i] = 0;
    if (threadIdx.x == 0) {
        s_bad = 0;
        s_max = 0;
    }
    __syncthreads();
    for (uint32_t s = threadIdx.x; s < cap; s += blockDim.x) {
        uint32_t L = lengths[s];
        if (L > 64) s_bad = 1;
        else if (L) {
            atomicAdd(&s_cnt[L], 1u);
            atomicMax(&s_max, L);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // Codebook.from_lengths validation (P/codebook.py:125-140)
        uint32_t used = 0;
        for (int L = 1; L <= 64; L++) used += s_cnt[L];
        int rc = 0;
        if (s_bad || used == 0) rc = 1;
        else if (used == 1) rc = (s_max != 1);
        else {
            int64_t avail = 1;
            for (int L = 1; L <= 64 && !rc; L++) {
                avail = 2 * avail - (int64_t)s_cnt[L];
                if (avail < 0 || avail > (int64_t)cap) rc = 1;
            }
            if (!rc && avail != 0) rc = 1;
        }
        if (rc) {
            set_status(st, LZB_E_CORRUPT);
            s_bad = 1;
        }
        uint64_t f = 0;
        uint32_t o = 0;
        for (int L = 1; L <= 64; L++) {
            f = (L == 1) ? 0 : (f + s_cnt[L - 1]) << 1;
            tab->first[L] = f;
            tab->cnt[L] = s_cnt[L];
            tab->off[L] = o;
            s_off[L] = o;
            o += s_cnt[L];
        }
        tab->first[0] = 0;
        tab->cnt[0] = 0;
        tab->off[0] = 0;
        tab->maxlen = s_max;
        tab->nsym = used;
        if (s_max > maxlen_hint) {
            set_status(st, LZB_E_CORRUPT);
            s_bad = 1;
        }
    }
    __syncthreads();
    if (s_bad) return;
    // symbols in (length, symbol) order + LUT fill; warp 0 ranks 32 symbols at a time
    if (threadIdx.x < 32) {
        const uint32_t lane = threadIdx.x;
        for (uint32_t s0 = 0; s0 < cap; s0 += 32) {
            uint32_t s = s0 + lane;
            uint32_t L = s < cap ? lengths[s] : 0u;
            uint32_t peers = __match_any_sync(0xffffffffu, L);
            uint32_t rank = __popc(peers & ((1u << lane) - 1u));
            uint32_t o = s_off[L];
            if (s < cap && L) syms[o + rank] = s;
            __syncwarp();
            if (L && lane == (uint32_t)(__ffs(peers) - 1)) s_off[L] = o + __popc(peers);
            __syncwarp();
        }
    }
    __syncthreads();
}

// LUTs over every 12-bit window, one window per thread: a single greedy pass
// decodes the complete code words inside the window (up to 12); every LUT
// variant is a prefix of that sequence.
__global__ void __launch_bounds__(1024) k_dec_luts(DecTables *tab, const uint32_t *syms, uint32_t cap,
                                                   lzb_dstatus *st) {
    __shared__ uint64_t s_first[65], s_cnt[65];
    __shared__ uint32_t s_off[65];
    for (uint32_t i = threadIdx.x; i < 65; i += blockDim.x) {
        s_first[i] = tab->first[i];
        s_cnt[i] = tab->cnt[i];
        s_off[i] = tab->off[i];
    }
    __syncthreads();
    if (st->code) return;
    const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= kLutSize) return;
    const uint32_t maxlen = tab->maxlen;
    const bool wide_cap = cap > 65536;  // symbols do not fit the u16 LUT fields
    uint32_t len[12], sym[12], n = 0, used = 0;
    while (n < 12) {
        uint32_t L = 0, sy = 0;
        for (uint32_t l = 1; l + used <= (uint32_t)kLutBits && l <= maxlen; l++) {
            const uint32_t code = (v >> (kLutBits - used - l)) & ((1u << l) - 1u);
            const uint64_t f = s_first[l], k = s_cnt[l];
            if (k && code >= f && code - f < k) {
                L = l;
                sy = wide_cap ? 0u : syms[s_off[l] + (uint32_t)(code - f)];
                break;
            }
        }
        if (!L) break;
        len[n] = L;
        sym[n] = sy;
        used += L;
        n++;
    }
    // lutm: up to three code words (count 0 for cap > 65536)
    {
        const uint32_t m = wide_cap ? 0u : (n < 3 ? n : 3u);
        uint64_t e = m;
        for (uint32_t i = 0; i < m; i++) {
            e |= (uint64_t)len[i] << (2 + 4 * i);
            e |= (uint64_t)sym[i] << (16 + 16 * i);
        }
        tab->lutm[v] = e;
    }
    // lut8: byte deltas against cap/2 - 128, the prefix whose symbols fit a byte
    {
        const int32_t base = (int32_t)(cap / 2) - 128;
        uint32_t m = wide_cap ? 0u : (n < 6 ? n : 6u);
        for (uint32_t i = 0; i < m; i++) {
            const int32_t d = (int32_t)sym[i] - base;
            if (d < 0 || d > 254) {  // 255 is the final pass's escape byte
                m = i;
                break;
            }
        }
        uint64_t e = 0;
        uint32_t u = 0, sm = 0;
        for (uint32_t i = 0; i < m; i++) {
            e |= (uint64_t)(uint32_t)((int32_t)sym[i] - base) << (8 * i);
            sm |= 1u << u;
            u += len[i];
        }
        tab->lut8[v] = e | ((uint64_t)m << 48) | ((uint64_t)u << 51);
        tab->lut8s[v] = (uint16_t)sm;
        tab->lut1s[v] = (uint16_t)(n && !wide_cap ? sym[0] : 0u);
    }
    // lutb: all complete code words (count-only), their starts
    {
        uint32_t u = 0, sm = 0;
        for (uint32_t i = 0; i < n; i++) {
            sm |= 1u << u;
            u += len[i];
        }
        tab->lutb[v] = n | (u << 4) | (sm << 8);
        tab->lutc[v] = n ? (u | (n << 16)) : 0x80000000u;
    }
    // lut1: first code word: its length if <= 12 bits, else 0x80 | the shortest
    // length of a code word with this 12-bit prefix, 0 = invalid prefix
    {
        uint32_t l1 = n ? len[0] : 0u;
        for (uint32_t L = kLutBits + 1; L <= maxlen && !l1; L++) {
            const uint64_t f = s_first[L], k = s_cnt[L];
            if (!k) continue;
            const uint32_t sh = L - kLutBits;
            if ((f >> sh) <= v && v <= ((f + (k - 1)) >> sh)) l1 = 0x80u | L;
        }
        tab->lut1[v] = (uint8_t)l1;
    }
    // lut6: the first six code words as u16 symbols
    {
        const uint32_t m = wide_cap ? 0u : (n < 6 ? n : 6u);
        uint32_t w[3] = {0, 0, 0}, u = 0;
        for (uint32_t i = 0; i < m; i++) {
            w[i >> 1] |= (sym[i] & 0xFFFFu) << (16 * (i & 1));
            u += len[i];
        }
        tab->lut6[v] = make_uint4(w[0], w[1], w[2], m | (u << 8));
    }
}

// Level-1/2 composition: thread per (group, phase).  in: n_in maps of P entries
// (32-bit or 64-bit packed (count << 8) | exit).
template <typename InT>
__global__ void k_dec_compose(const InT *in, uint64_t n_in, uint32_t P, uint32_t G, uint64_t *out,
                              uint64_t nout, const unsigned int *nonuni) {
    if (*nonuni == 0) return;  // the uniform scan resolves the entries
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nout * P;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t g = i / P;
        uint32_t ph = (uint32_t)(i - g * P);
        uint64_t cnt = 0;
        uint32_t e = ph;
        uint64_t a = g * G, b = umin64(a + G, n_in);
        for (uint64_t k = a; k < b; k++) {
            uint64_t v = in[k * P + e];
            uint32_t ex = (uint32_t)(v & 0xFF);
            cnt += v >> 8;
            e = ex;
            if (ex == kExitInvalid || ex == kExitEnd) {
                // END is only legal as the very last map of the stream
                if (ex == kExitEnd && k + 1 != n_in) e = kExitInvalid;
                break;
            }
        }
        out[i] = (cnt << 8) | e;
    }
}

// Walk `n` maps of group `g` from entry phase e0 / offset o0, writing each
// member's entry + offset (used top-down).
template <typename InT>
__device__ __forceinline__ void walk_down(const InT *maps, uint32_t P, uint64_t a, uint64_t b,
                                          uint32_t e, uint64_t o, uint8_t *ent, uint64_t *off) {
    for (uint64_t k = a; k < b; k++) {
        ent[k] = (uint8_t)e;
        off[k] = o;
        if (e == kExitInvalid || e == kExitEnd) {
            e = kExitInvalid;
            continue;
        }
        uint64_t v = maps[k * P + e];
        o += v >> 8;
        e = (uint32_t)(v & 0xFF);
    }
}

// Fast composition.  When every subsequence's valid entry phases all exit
// at the same phase (they joined the chain -- the normal case for Huffman
// codes), subsequence t's entry is t-1's common exit no matter where t-1 was
// entered, so entries are direct and offsets one exclusive scan of the
// entered maps' counts (single pass, decoupled look-back).  Otherwise the
// hierarchical composition below runs instead.
__global__ void __launch_bounds__(256) k_dec_scan_uniform(DecParams p) {
    if (*p.nonuni != 0) return;
    __shared__ uint64_t s_t, s_ex;
    __shared__ uint64_t s_scan[33];
    __shared__ int s_bad;
    const uint64_t ntl = (p.T + 2047) / 2048;
    while (true) {
        if (threadIdx.x == 0) {
            s_t = atomicAdd(p.uticket, 1u);
            s_bad = 0;
        }
        __syncthreads();
        const uint64_t tl = s_t;
        if (tl >= ntl) break;
        const uint64_t b0 = tl * 2048 + (uint64_t)threadIdx.x * 8;
        uint64_t c[8], sum = 0;
        uint32_t ent[8];
        bool bad = false;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const uint64_t t = b0 + k;
            c[k] = 0;
            ent[k] = 0;
            if (t < p.T) {
                const uint32_t e = t == 0 ? p.entry0 : p.uexit[t - 1];
                ent[k] = e;
                if (e >= p.P || (t + 1 < p.T && p.uexit[t] == kExitEnd)) {
                    bad = true;  // no valid entry, or END before the last subsequence
                } else {
                    const uint32_t v = p.maps[t * p.P + e];
                    if ((v & 0xFF) == kExitInvalid) bad = true;
                    c[k] = v >> 8;
                }
                sum += c[k];
            }
        }
        if (bad) s_bad = 1;
        uint64_t tot;
        const uint64_t off = block_exclusive_scan<uint64_t>(sum, s_scan, &tot);
        if ((threadIdx.x >> 5) == 0) {
            const uint64_t ex = lookback_warp(p.ulb, tl, tot);
            if (lane_id() == 0) s_ex = ex;
        }
        __syncthreads();
        uint64_t run = s_ex + off;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const uint64_t t = b0 + k;
            if (t < p.T) {
                p.ent0[t] = (uint8_t)ent[k];
                p.off0[t] = run;
            }
            run += c[k];
        }
        if (s_bad) set_status(p.st, LZB_E_CORRUPT);
        if (tl == ntl - 1 && threadIdx.x == 0) {
            const uint64_t total = s_ex + tot;
            if (p.uexit[p.T - 1] != p.exit_expect || total != p.count) set_status(p.st, LZB_E_CORRUPT);
            p.st->u[0] = total;
        }
        __syncthreads();
    }
}

__global__ void k_dec_top(DecParams p) {
    if (*p.nonuni == 0) return;
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    uint32_t e = p.entry0;
    uint64_t o = 0;
    for (uint64_t h = 0; h < p.ng2; h++) {
        p.ent2[h] = (uint8_t)e;
        p.off2[h] = o;
        if (e == kExitInvalid || e == kExitEnd) {
            e = kExitInvalid;
            continue;
        }
        uint64_t v = p.g2[h * p.P + e];
        o += v >> 8;
        e = (uint32_t)(v & 0xFF);
    }
    if (e != p.exit_expect || o != p.count) set_status(p.st, LZB_E_CORRUPT);
    p.st->u[0] = o;
}

__global__ void k_dec_down2(DecParams p) {
    if (*p.nonuni == 0) return;
    for (uint64_t h = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; h < p.ng2;
         h += (uint64_t)gridDim.x * blockDim.x)
        walk_down(p.g1, p.P, h * p.G, umin64(h * p.G + p.G, p.ng1), p.ent2[h], p.off2[h], p.ent1,
                  p.off1);
}

__global__ void k_dec_down1(DecParams p) {
    if (*p.nonuni == 0) return;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < p.ng1;
         g += (uint64_t)gridDim.x * blockDim.x)
        walk_down(p.maps, p.P, g * p.G, umin64(g * p.G + p.G, p.T), p.ent1[g], p.off1[g], p.ent0,
                  p.off0);
}

// Final decode: lanes decode their subsequence from the resolved entry,
// up to three symbols per LUT lookup, staged 32 per round in shared memory;
// the warp then writes each lane's run cooperatively (coalesced).
constexpr int kFThreads = 512;
constexpr int kStage = 32;
template <typename SymT>
__global__ void __launch_bounds__(kFThreads) k_dec_final(DecParams p) {
    extern __shared__ __align__(16) unsigned char f_smem[];
    uint64_t *s_lut = reinterpret_cast<uint64_t *>(f_smem);
    typedef SymT StageRow[kStage + 1];
    StageRow(*s_stage)[32] = reinterpret_cast<StageRow(*)[32]>(f_smem + kLutSize * sizeof(uint64_t));
    __shared__ DecCanon s_can;
    for (uint32_t i = threadIdx.x; i < kLutSize; i += blockDim.x) s_lut[i] = p.tab->lutm[i];
    load_canon(s_can, p.tab);
    __syncthreads();
    if (p.st->code) return;  // corrupt stream: leave the output untouched
    const DecCanon *tab = &s_can;
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    SymT *out = static_cast<SymT *>(p.out);
    SymT *stg = &s_stage[warp][lane][0];
    const uint64_t tstride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t tb = blockIdx.x * (uint64_t)blockDim.x + (threadIdx.x & ~31u); tb < p.T;
         tb += tstride) {
        const uint64_t t = tb + lane;
        const bool act = t < p.T;
        Win r;
        uint64_t o = 0, t0 = 0;
        uint32_t rel = 0, stop = 0;
        bool live = false;
        if (act) {
            const uint32_t e = p.ent0[t];
            if (e != kExitInvalid && e != kExitEnd) {
                t0 = t * p.S;
                stop = (uint32_t)(((t == p.T - 1) ? p.bit_len : umin64(t0 + p.S, p.bit_len)) - t0);
                rel = e;
                r.init(p, t0 + rel);
                o = p.off0[t];
                live = rel < stop;
            }
        }
        const uint32_t lim = stop >= (uint32_t)kLutBits ? stop - kLutBits : 0;
        while (__any_sync(0xffffffffu, live)) {
            uint32_t k = 0;
            // lock-step round: every lane takes one step per iteration (the
            // vote re-converges the warp), at most kStage symbols per lane
            bool go = live;
            while (__any_sync(0xffffffffu, go)) {
                if (go) {
                    const uint64_t e = s_lut[r.peek12()];
                    const uint32_t n = lm_count(e);
                    if (n && k <= (uint32_t)kStage - 3 && rel + kLutBits <= stop) {
                        stg[k] = (SymT)lm_sym(e, 0);
                        stg[k + 1] = (SymT)lm_sym(e, 1);
                        stg[k + 2] = (SymT)lm_sym(e, 2);
                        const uint32_t used = lm_len(e, 0) + lm_len(e, 1) + lm_len(e, 2);
                        r.consume(p, used);
                        rel += used;
                        k += n;
                    } else {
                        uint32_t L, sym;
                        if (n) {
                            L = lm_len(e, 0);
                            sym = lm_sym(e, 0);
                        } else {
                            L = decode_long(p, tab, t0 + rel, sym);
                        }
                        if (L == 0) {
                            rel = stop;
                        } else {
                            stg[k++] = (SymT)sym;
                            if (L <= 32) r.consume(p, L);
                            else r.init(p, t0 + rel + L);
                            rel += L;
                        }
                    }
                    go = rel < stop && k < (uint32_t)kStage;
                }
            }
            live = rel < stop;
            __syncwarp();
            // cooperative write-out of every lane's k symbols
            for (uint32_t j = 0; j < 32; j++) {
                const uint32_t kj = __shfl_sync(0xffffffffu, k, j);
                const uint64_t oj = __shfl_sync(0xffffffffu, o, j);
                if (lane < kj && oj + lane < p.count) out[oj + lane] = s_stage[warp][j][lane];
            }
            o += k;
            __syncwarp();
        }
    }
}

#include "lzb_dec3.cuh"

// ----------------------------------------------------------------------------
struct DecLayout {
    uint32_t S, P, G;
    uint64_t T, ng1, ng2;
};

static DecLayout dec_layout(uint64_t bit_len, uint32_t maxlen) {
    DecLayout L;
    L.P = maxlen < 1 ? 1 : maxlen;
    L.S = kS3;  // one warp per subsequence, one lane per 128-bit microblock (lzb_dec3.cuh)
    L.T = bit_len ? (bit_len + L.S - 1) / L.S : 1;
    L.G = 256;
    L.ng1 = (L.T + L.G - 1) / L.G;
    L.ng2 = (L.ng1 + L.G - 1) / L.G;
    return L;
}

template <typename Sc>
static void dec_scratch(Sc &s, const DecLayout &L, uint32_t cap) {
    s.template take<DecTables>(1);
    s.template take<uint32_t>(cap);
    s.template take<uint32_t>(L.T * L.P);
    s.template take<uint64_t>(L.ng1 * L.P);
    s.template take<uint64_t>(L.ng2 * L.P);
    s.template take<uint8_t>(L.ng2);
    s.template take<uint64_t>(L.ng2);
    s.template take<uint8_t>(L.ng1);
    s.template take<uint64_t>(L.ng1);
    s.template take<uint8_t>(L.T);
    s.template take<uint64_t>(L.T);
    s.template take<uint16_t>(L.T * 32);
    s.template take<uint64_t>(L.T);
    s.template take<uint8_t>(L.T);
    s.template take<unsigned int>(4);
    s.template take<uint64_t>(L.T / 2048 + 2);
}

static int dev_sms() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms > 0 ? sms : 148;
}

// ---- K5 v4 plan (lzb_dec4.cuh) ----
// scratch order: tables, syms, cp, soff, sbm, srest, sx0, sexit, look-back + ticket
static void d4_sizes(ScratchSize &sc, uint64_t T, uint32_t cap) {
    const uint64_t ntl = (T + kD4ResolveThreads - 1) / kD4ResolveThreads;
    sc.take<DecTables>(1);
    sc.take<uint32_t>(cap);
    sc.take<uint16_t>(32 * T);
    sc.take<uint64_t>(T);
    sc.take<uint64_t>(T);
    sc.take<uint32_t>(T);
    sc.take<uint8_t>(T);
    sc.take<uint8_t>(T);
    sc.take<uint8_t>(T);
    sc.take<uint64_t>(ntl + 2);
}

static bool d4_take(Scratch &sc, uint64_t T, uint32_t cap, D4Plan &p) {
    const uint64_t ntl = (T + kD4ResolveThreads - 1) / kD4ResolveThreads;
    p.tab = sc.take<DecTables>(1);
    p.syms = sc.take<uint32_t>(cap);
    p.cp = sc.take<uint16_t>(32 * T);
    p.soff = sc.take<uint64_t>(T);
    p.sbm = sc.take<uint64_t>(T);
    p.srest = sc.take<uint32_t>(T);
    p.sx0 = sc.take<uint8_t>(T);
    p.sexit = sc.take<uint8_t>(T);
    p.sirr = sc.take<uint8_t>(T);
    p.lb = sc.take<uint64_t>(ntl + 2);  // + the ticket word (one memset)
    p.ticket = p.lb ? reinterpret_cast<unsigned int *>(p.lb + ntl + 1) : nullptr;
    return p.ticket != nullptr;
}

size_t d4_scratch_bytes(uint64_t bit_len, uint64_t count, uint32_t cap) {
    ScratchSize s;
    const uint64_t T = bit_len ? (bit_len + kD4S - 1) / kD4S : 1;
    (void)count;
    d4_sizes(s, T, cap);
    return s.bytes();
}

int d4_plan(const uint8_t *bits, uint32_t bit_phase, uint64_t bit_len, uint64_t count,
            const uint8_t *lengths, uint32_t cap, uint32_t maxlen, lzb_dstatus *st, Scratch &sc,
            cudaStream_t s, D4Plan &p) {
    if (!bits || bit_len == 0 || count == 0) return LZB_E_ARG;
    p.bit_len = bit_len;
    p.count = count;
    p.T = (bit_len + kD4S - 1) / kD4S;
    p.nmb = (bit_len + kD4MB - 1) / kD4MB;
    if (!d4_take(sc, p.T, cap, p)) return LZB_E_ARG;
    uintptr_t a = reinterpret_cast<uintptr_t>(bits);
    p.words = reinterpret_cast<const uint32_t *>(a & ~uintptr_t(3));
    p.head = (uint32_t)(a & 3) * 8 + bit_phase;
    p.nwords = ((p.head + bit_len + 7) / 8 + 3) / 4;
    p.base8 = (int32_t)(cap / 2) - 128;
    p.st = st;
    const uint64_t ntl = (p.T + kD4ResolveThreads - 1) / kD4ResolveThreads;
    LZB_CUDA_TRY(cudaMemsetAsync(p.lb, 0, (ntl + 2) * sizeof(uint64_t), s));
    k_dec_tables<<<1, 1024, 0, s>>>(lengths, cap, maxlen, const_cast<DecTables *>(p.tab),
                                    const_cast<uint32_t *>(p.syms), st);
    LZB_LAUNCH_CHECK();
    k_dec_luts<<<kLutSize / 1024, 1024, 0, s>>>(const_cast<DecTables *>(p.tab), p.syms, cap, st);
    LZB_LAUNCH_CHECK();
    const int sms = dev_sms();
    // 32 CTAs per SM requested, ~5 resident: later CTAs fill in behind the
    // slow subsequences (measured: 8 / 16 / 32 / 64 per SM -> K5 3.67 / 3.61 /
    // 3.59 / 3.58 ms on C5q, C3 5.09 -> 4.94 ms at 32; sized to the resident
    // CTAs exactly: 3.77 ms)
    k_dec4_count<<<(unsigned)umin64((p.T + kD4Warps - 1) / kD4Warps, (uint64_t)sms * 32), kD4Warps * 32, 0, s>>>(p);
    LZB_LAUNCH_CHECK();
    k_dec4_resolve<<<(unsigned)umin64(ntl, (uint64_t)sms * 4), kD4ResolveThreads, 0, s>>>(p);
    LZB_LAUNCH_CHECK();
    return LZB_OK;
}

}  // namespace lzb

using namespace lzb;

// ---------------------------------------------------------------------------
extern "C" size_t lzb_huff_encode_scratch_bytes(uint64_t n) {
    ScratchSize s;
    uint64_t nt = (n + kETile - 1) / kETile;
    s.take<uint64_t>(nt ? nt : 1);
    s.take<unsigned int>(4);
    s.take<uint64_t>(4 * (nt ? nt : 1));
    ScratchSize w;  // warp-tile path
    uint64_t ntw = (n + kWTile - 1) / kWTile;
    w.take<uint32_t>(ntw + 1);
    w.take<uint16_t>(32 * (ntw ? ntw : 1));
    w.take<uint64_t>(ntw + 1);
    w.take<uint64_t>((ntw + 1 + 2047) / 2048 + 1);
    w.take<unsigned int>(4);
    w.take<uint32_t>(2 * (ntw ? ntw : 1));
    return s.bytes() > w.bytes() ? s.bytes() : w.bytes();
}

static int huff_encode_w(const void *sym, uint64_t n, const uint8_t *lengths, const uint64_t *codes,
                         uint32_t cap, uint32_t maxlen, uint8_t *out, uint64_t bit_offset,
                         lzb_dstatus *st, void *scratch, size_t scratch_bytes, cudaStream_t s) {
    const uint64_t ntw = (n + kWTile - 1) / kWTile;
    Scratch sc(scratch, scratch_bytes);
    EncWParams p;
    const uint64_t nscan = (ntw + 1 + 2047) / 2048;
    p.cnt = sc.take<uint32_t>(ntw + 1);
    p.lcnt = sc.take<uint16_t>(32 * ntw);
    p.toff = sc.take<uint64_t>(ntw + 1);
    p.lb = sc.take<uint64_t>(nscan + 1);
    p.ticket = sc.take<unsigned int>(4);
    p.frag = sc.take<uint32_t>(2 * ntw);
    if (!p.frag) return LZB_E_ARG;
    LZB_CUDA_TRY(cudaMemsetAsync(p.lb, 0, (nscan + 1) * sizeof(uint64_t), s));
    LZB_CUDA_TRY(cudaMemsetAsync(p.ticket, 0, 4 * sizeof(unsigned int), s));
    LZB_CUDA_TRY(cudaMemsetAsync(p.cnt + ntw, 0, sizeof(uint32_t), s));
    p.sym = static_cast<const uint16_t *>(sym);
    p.n = n;
    p.lengths = lengths;
    p.codes = codes;
    p.cap = cap;
    p.out = out;
    p.bit_offset = bit_offset;
    p.st = st;
    p.ntiles = ntw;
    p.wwords = (32 * maxlen + 2 + 3) & ~3u;
    const size_t smem = (((size_t)cap * 8 + 15) & ~(size_t)15) + (size_t)kWWarps * kWTile * 2 +
                        (size_t)kWWarps * p.wwords * 4;
    LZB_CUDA_TRY(set_dyn_smem(k_huff_encode_w, smem));
    int per_sm = 0;
    LZB_CUDA_TRY(occupancy(&per_sm, k_huff_encode_w, kWWarps * 32, smem));
    if (per_sm < 1) return LZB_E_ARG;
    // 4x the resident CTAs: the later waves even out the warps' tile loads
    // (C5q encode 1.47 -> 1.40 ms; count pass likewise at 32 CTAs per SM)
    uint64_t grid = (uint64_t)dev_sms() * per_sm * 4;
    const uint64_t need = (ntw + kWWarps - 1) / kWWarps;
    if (grid > need) grid = need;
    const int sms = dev_sms();
    k_huff_count_w<<<(unsigned)umin64((ntw + 7) / 8, (uint64_t)sms * 32), 256, 0, s>>>(p);
    LZB_LAUNCH_CHECK();
    k_huff_scan_w<<<(unsigned)nscan, 256, 0, s>>>(p);
    LZB_LAUNCH_CHECK();
    k_huff_encode_w<<<(unsigned)grid, kWWarps * 32, smem, s>>>(p);
    LZB_LAUNCH_CHECK();
    k_huff_fixup_w<<<(unsigned)umin64((ntw + 255) / 256, 4096), 256, 0, s>>>(p);
    LZB_LAUNCH_CHECK();
    return LZB_OK;
}

static int huff_encode_impl(const void *sym, int sym_bytes, uint64_t n, const uint8_t *lengths,
                            const uint64_t *codes, uint32_t cap, uint32_t maxlen, uint8_t *out,
                            uint64_t out_bytes, uint64_t bit_offset, lzb_dstatus *st, void *scratch,
                            size_t scratch_bytes, void *stream) {
    if (!lengths || !codes || !st || (sym_bytes != 2 && sym_bytes != 4) || cap == 0)
        return LZB_E_ARG;
    cudaStream_t s = as_stream(stream);
    LZB_CUDA_TRY(cudaMemsetAsync(st, 0, sizeof(lzb_dstatus), s));
    if (n == 0) return LZB_OK;
    if (!sym || !out) return LZB_E_ARG;
    const bool wpath = sym_bytes == 2 && cap <= 4096 && (reinterpret_cast<uintptr_t>(sym) & 1) == 0;
    if (maxlen == LZB_MAXLEN_DEVICE) {  // book built on the device: the 32-bit path, sized for 32
        if (!wpath) return LZB_E_ARG;
        return huff_encode_w(sym, n, lengths, codes, cap, 32, out, bit_offset, st, scratch, scratch_bytes, s);
    }
    if (wpath && maxlen >= 1 && maxlen <= 32)
        return huff_encode_w(sym, n, lengths, codes, cap, maxlen, out, bit_offset, st, scratch,
                             scratch_bytes, s);
    uint64_t nt = (n + kETile - 1) / kETile;
    Scratch sc(scratch, scratch_bytes);
    EncParams p;
    p.lb = sc.take<uint64_t>(nt);
    p.ticket = sc.take<unsigned int>(4);
    p.frag = sc.take<uint64_t>(4 * nt);
    if (!p.frag) return LZB_E_ARG;
    LZB_CUDA_TRY(cudaMemsetAsync(p.lb, 0, nt * sizeof(uint64_t), s));
    LZB_CUDA_TRY(cudaMemsetAsync(p.ticket, 0, 4 * sizeof(unsigned int), s));
    p.sym = sym;
    p.n = n;
    p.lengths = lengths;
    p.codes = codes;
    p.cap = cap;
    p.out = out;
    p.out_bytes = out_bytes;
    p.bit_offset = bit_offset;
    p.st = st;
    p.ntiles = nt;
    p.maxlen = (maxlen >= 1 && maxlen <= 64) ? maxlen : 64;
    p.table_smem = cap <= 4096;
    const bool shortc = p.maxlen <= 32;
    size_t table = p.table_smem ? align_up((size_t)cap * 9, 16) : 0;
    size_t smem = table + ((size_t)kETile * p.maxlen / 32 + 4) * sizeof(uint32_t);
    void (*kern)(EncParams);
    if (sym_bytes == 2) {
        if (shortc) kern = p.table_smem ? k_huff_encode<uint16_t, true, true> : k_huff_encode<uint16_t, true, false>;
        else kern = p.table_smem ? k_huff_encode<uint16_t, false, true> : k_huff_encode<uint16_t, false, false>;
    } else {
        if (shortc) kern = p.table_smem ? k_huff_encode<uint32_t, true, true> : k_huff_encode<uint32_t, true, false>;
        else kern = p.table_smem ? k_huff_encode<uint32_t, false, true> : k_huff_encode<uint32_t, false, false>;
    }
    LZB_CUDA_TRY(set_dyn_smem(kern, smem));
    int per_sm = 0;
    LZB_CUDA_TRY(occupancy(&per_sm, kern, kEThreads, smem));
    uint64_t grid = (uint64_t)dev_sms() * (per_sm > 0 ? per_sm : 1);
    if (grid > nt) grid = nt;
    kern<<<(unsigned)grid, kEThreads, smem, s>>>(p);
    LZB_LAUNCH_CHECK();
    // bytes actually owned by this stream: through the last bit
    k_huff_fixup<<<(unsigned)umin64((nt + 255) / 256, 4096), 256, 0, s>>>(p);
    LZB_LAUNCH_CHECK();
    return LZB_OK;
}

extern "C" int lzb_huff_encode(const void *sym, int sym_bytes, uint64_t n, const uint8_t *lengths,
                               const uint64_t *codes, uint32_t cap, uint32_t maxlen, uint8_t *out,
                               uint64_t out_bytes, lzb_dstatus *st, void *scratch,
                               size_t scratch_bytes, void *stream) {
    return huff_encode_impl(sym, sym_bytes, n, lengths, codes, cap, maxlen, out, out_bytes, 0, st,
                            scratch, scratch_bytes, stream);
}

// Multi-GPU slab variant: the slab's first bit lands at bit `bit_offset` (0..7)
// of out[0]; out[0]'s leading bits and the last byte's trailing bits are left
// zero for an OR-merge with the neighbouring slabs.
extern "C" int lzb_huff_encode_at(const void *sym, int sym_bytes, uint64_t n, const uint8_t *lengths,
                                  const uint64_t *codes, uint32_t cap, uint32_t maxlen,
                                  uint64_t bit_offset, uint8_t *out, uint64_t out_bytes,
                                  lzb_dstatus *st, void *scratch, size_t scratch_bytes, void *stream) {
    if (bit_offset > 7) return LZB_E_ARG;
    return huff_encode_impl(sym, sym_bytes, n, lengths, codes, cap, maxlen, out, out_bytes,
                            bit_offset, st, scratch, scratch_bytes, stream);
}

extern "C" size_t lzb_huff_decode_scratch_bytes(uint64_t bit_len, uint32_t maxlen, uint32_t cap) {
    ScratchSize s;
    dec_scratch(s, dec_layout(bit_len, maxlen), cap);
    // the fast path's plan is sized by symbols too; a stream of bit_len bits
    // holds at most bit_len code words
    const size_t f = d4_scratch_bytes(bit_len, bit_len, cap);
    return s.bytes() > f ? s.bytes() : f;
}

// Tables + LUTs + the scratch carve-up shared by the whole-stream and the
// bit-range entry points.  `bits`/`bit_phase` locate the first bit to decode,
// `bit_len` bits are decoded, code words may read up to `total_bits`.
static int dec_setup(const uint8_t *bits, uint32_t bit_phase, uint64_t bit_len, uint64_t total_bits,
                     uint64_t count, const uint8_t *lengths, uint32_t cap, uint32_t maxlen, void *sym,
                     lzb_dstatus *st, void *scratch, size_t scratch_bytes, cudaStream_t s, bool tables,
                     DecParams &p, DecLayout &L) {
    L = dec_layout(bit_len, maxlen);
    Scratch sc(scratch, scratch_bytes);
    DecTables *tab = sc.take<DecTables>(1);
    uint32_t *syms = sc.take<uint32_t>(cap);
    if (!syms) return LZB_E_ARG;
    if (tables) {
        k_dec_tables<<<1, 1024, 0, s>>>(lengths, cap, maxlen, tab, syms, st);
        LZB_LAUNCH_CHECK();
        k_dec_luts<<<kLutSize / 1024, 1024, 0, s>>>(tab, syms, cap, st);
        LZB_LAUNCH_CHECK();
    }
    uintptr_t a = reinterpret_cast<uintptr_t>(bits);
    p.words = reinterpret_cast<const uint32_t *>(a & ~uintptr_t(3));
    p.head = (uint32_t)(a & 3) * 8 + bit_phase;
    p.nwords = ((p.head + total_bits + 7) / 8 + 3) / 4;
    p.bit_len = bit_len;
    p.total_bits = total_bits;
    p.count = count;
    p.entry0 = 0;
    p.exit_expect = kExitEnd;
    p.open_end = 0;
    p.tab = tab;
    p.syms = syms;
    p.psoff = nullptr;
    p.pirr = nullptr;
    p.S = L.S;
    p.T = L.T;
    p.P = L.P;
    p.G = L.G;
    p.ng1 = L.ng1;
    p.ng2 = L.ng2;
    p.maps = sc.take<uint32_t>(L.T * L.P);
    p.g1 = sc.take<uint64_t>(L.ng1 * L.P);
    p.g2 = sc.take<uint64_t>(L.ng2 * L.P);
    p.ent2 = sc.take<uint8_t>(L.ng2);
    p.off2 = sc.take<uint64_t>(L.ng2);
    p.ent1 = sc.take<uint8_t>(L.ng1);
    p.off1 = sc.take<uint64_t>(L.ng1);
    p.ent0 = sc.take<uint8_t>(L.T);
    p.off0 = sc.take<uint64_t>(L.T);
    p.cp = sc.take<uint16_t>(L.T * 32);
    p.irr = sc.take<uint64_t>(L.T);
    p.uexit = sc.take<uint8_t>(L.T);
    p.nonuni = sc.take<unsigned int>(4);
    p.uticket = p.nonuni + 1;  // nonuni[2]: an always-set gate for the range composition
    p.ulb = sc.take<uint64_t>(L.T / 2048 + 2);
    if (!p.ulb) return LZB_E_ARG;
    p.st = st;
    p.out = sym;
    return LZB_OK;
}

// Per-subsequence transfer maps (phases >= the book's real max length cannot
// be entries: P = maxlen hint, k_dec_tables flags a hint that disagrees with
// the lengths as corrupt), then the uniform-exit scan.
static int dec_maps(DecParams &p, const DecLayout &L, cudaStream_t s) {
    const int sms = dev_sms();
    LZB_CUDA_TRY(cudaMemsetAsync(p.nonuni, 0, 4 * sizeof(unsigned int), s));
    k_dec_maps3<<<(unsigned)umin64((L.T + kD3Warps - 1) / kD3Warps, (uint64_t)sms * 16), kD3Warps * 32, 0, s>>>(p);
    LZB_LAUNCH_CHECK();
    return LZB_OK;
}

static int dec_compose(DecParams &p, const DecLayout &L, cudaStream_t s, const unsigned int *gate) {
    const int sms = dev_sms();
    k_dec_compose<uint32_t><<<(unsigned)umin64((L.ng1 * L.P + 255) / 256, (uint64_t)sms * 32), 256, 0, s>>>(
        p.maps, L.T, L.P, L.G, p.g1, L.ng1, gate);
    LZB_LAUNCH_CHECK();
    k_dec_compose<uint64_t><<<(unsigned)umin64((L.ng2 * L.P + 255) / 256, (uint64_t)sms * 32), 256, 0, s>>>(
        p.g1, L.ng1, L.P, L.G, p.g2, L.ng2, gate);
    LZB_LAUNCH_CHECK();
    return LZB_OK;
}

// Entry phase + symbol offset of every subsequence (uniform scan, or the
// composed hierarchy top-down), then the final decode into p.out.
static int dec_resolve_final(DecParams &p, const DecLayout &L, cudaStream_t s, int sym_bytes, uint32_t cap) {
    const int sms = dev_sms();
    LZB_CUDA_TRY(cudaMemsetAsync(p.uticket, 0, sizeof(unsigned int), s));
    LZB_CUDA_TRY(cudaMemsetAsync(p.ulb, 0, (L.T / 2048 + 2) * sizeof(uint64_t), s));
    k_dec_scan_uniform<<<(unsigned)umin64((L.T + 2047) / 2048, (uint64_t)sms * 4), 256, 0, s>>>(p);
    LZB_LAUNCH_CHECK();
    k_dec_top<<<1, 32, 0, s>>>(p);
    LZB_LAUNCH_CHECK();
    k_dec_down2<<<(unsigned)umin64((L.ng2 + 127) / 128, 1024), 128, 0, s>>>(p);
    LZB_LAUNCH_CHECK();
    k_dec_down1<<<(unsigned)umin64((L.ng1 + 127) / 128, (uint64_t)sms * 8), 128, 0, s>>>(p);
    LZB_LAUNCH_CHECK();
    if (sym_bytes == 2 && cap <= 65536) {
        const size_t f9 = (size_t)kLutSize * (8 + 2 + 2 + 1) + (size_t)kF9Warps * kF9Stage +
                          (size_t)kF9Warps * 2 * kStgWords * 4;
        LZB_CUDA_TRY(set_dyn_smem(k_dec_final9, f9));
        const unsigned g9 = (unsigned)umin64((L.T + kF9Warps - 1) / kF9Warps, (uint64_t)sms);
        k_dec_final9<<<g9, kF9Warps * 32, f9, s>>>(p, cap);
    } else {
        const unsigned fg = (unsigned)umin64((L.T + kFThreads - 1) / kFThreads, (uint64_t)sms * 4);
        const size_t fsm = kLutSize * sizeof(uint64_t) + (size_t)(kFThreads / 32) * 32 * (kStage + 1) * sym_bytes;
        auto kern = sym_bytes == 2 ? k_dec_final<uint16_t> : k_dec_final<uint32_t>;
        LZB_CUDA_TRY(set_dyn_smem(kern, fsm));
        kern<<<fg, kFThreads, fsm, s>>>(p);
    }
    LZB_LAUNCH_CHECK();
    return LZB_OK;
}

static int huff_decode_impl(const uint8_t *bits, uint32_t bit_phase, uint64_t bit_len, uint64_t count,
                            const uint8_t *lengths, uint32_t cap, uint32_t maxlen, void *sym, int sym_bytes,
                            lzb_dstatus *st, void *scratch, size_t scratch_bytes, void *stream) {
    if (!lengths || !st || (sym_bytes != 2 && sym_bytes != 4) || cap == 0 || maxlen == 0 ||
        maxlen > 64 || bit_phase > 7)
        return LZB_E_ARG;
    cudaStream_t s = as_stream(stream);
    LZB_CUDA_TRY(cudaMemsetAsync(st, 0, sizeof(lzb_dstatus), s));
    if (count == 0) {
        // P/huffman.py:114-117: tables are still validated
        Scratch sc(scratch, scratch_bytes);
        DecTables *tab = sc.take<DecTables>(1);
        uint32_t *syms = sc.take<uint32_t>(cap);
        if (!syms) return LZB_E_ARG;
        k_dec_tables<<<1, 1024, 0, s>>>(lengths, cap, maxlen, tab, syms, st);
        LZB_LAUNCH_CHECK();
        if (bit_len != 0) {
            lzb_dstatus h{};
            h.code = LZB_E_CORRUPT;
            LZB_CUDA_TRY(cudaMemcpyAsync(st, &h, sizeof(int32_t), cudaMemcpyHostToDevice, s));
            LZB_CUDA_TRY(cudaStreamSynchronize(s));
        }
        return LZB_OK;
    }
    if (!bits || !sym) return LZB_E_ARG;
    DecParams p;
    DecLayout L;
    int rc = dec_setup(bits, bit_phase, bit_len, bit_len, count, lengths, cap, maxlen, sym, st, scratch,
                       scratch_bytes, s, true, p, L);
    if (rc != LZB_OK) return rc;
    if ((rc = dec_maps(p, L, s)) != LZB_OK) return rc;
    if ((rc = dec_compose(p, L, s, p.nonuni)) != LZB_OK) return rc;
    return dec_resolve_final(p, L, s, sym_bytes, cap);
}

// Fast path (K5 v4, lzb_dec4.cuh) for u16 symbols; LZB_E_RETRY in st sends the
// caller to lzb_huff_decode_robust.
extern "C" int lzb_huff_decode(const uint8_t *bits, uint64_t bit_len, uint64_t count,
                               const uint8_t *lengths, uint32_t cap, uint32_t maxlen, void *sym,
                               int sym_bytes, lzb_dstatus *st, void *scratch, size_t scratch_bytes,
                               void *stream) {
    if (sym_bytes != 2 || cap > 65536 || count == 0 || bit_len == 0 || !bits || !sym || !lengths || !st ||
        maxlen == 0 || maxlen > 64 || (reinterpret_cast<uintptr_t>(sym) & 1))
        return huff_decode_impl(bits, 0, bit_len, count, lengths, cap, maxlen, sym, sym_bytes, st, scratch,
                                scratch_bytes, stream);
    cudaStream_t s = as_stream(stream);
    LZB_CUDA_TRY(cudaMemsetAsync(st, 0, sizeof(lzb_dstatus), s));
    Scratch sc(scratch, scratch_bytes);
    D4Plan p;
    int rc = d4_plan(bits, 0, bit_len, count, lengths, cap, maxlen, st, sc, s, p);
    if (rc != LZB_OK) return rc;
    // final decode: k_dec_final9 (warp per subsequence, byte stage, coalesced
    // u16 stores) reading the entries and offsets of the plan
    DecParams q{};
    q.words = p.words;
    q.head = p.head;
    q.nwords = p.nwords;
    q.bit_len = bit_len;
    q.total_bits = bit_len;
    q.count = count;
    q.tab = p.tab;
    q.syms = p.syms;
    q.S = kS3;
    q.T = p.T;
    q.P = maxlen;
    q.cp = p.cp;
    q.psoff = p.soff;
    q.pirr = p.sirr;
    q.st = st;
    q.out = sym;
    q.entry0 = 0;
    q.exit_expect = kExitEnd;
    q.open_end = 0;
    const int sms = dev_sms();
    const size_t f9 = (size_t)kLutSize * (8 + 2 + 2 + 1) + (size_t)kF9Warps * kF9Stage +
                      (size_t)kF9Warps * 2 * kStgWords * 4;
    LZB_CUDA_TRY(set_dyn_smem(k_dec_final9, f9));
    const unsigned g9 = (unsigned)umin64((p.T + kF9Warps - 1) / kF9Warps, (uint64_t)sms);
    k_dec_final9<<<g9, kF9Warps * 32, f9, s>>>(q, cap);
    LZB_LAUNCH_CHECK();
    return LZB_OK;
}

// The exhaustive decoder: transfer maps of every entry phase composed over the
// whole stream (any prefix code, also books that never resynchronise).
extern "C" int lzb_huff_decode_robust(const uint8_t *bits, uint64_t bit_len, uint64_t count,
                                      const uint8_t *lengths, uint32_t cap, uint32_t maxlen, void *sym,
                                      int sym_bytes, lzb_dstatus *st, void *scratch, size_t scratch_bytes,
                                      void *stream) {
    return huff_decode_impl(bits, 0, bit_len, count, lengths, cap, maxlen, sym, sym_bytes, st, scratch,
                            scratch_bytes, stream);
}

extern "C" int lzb_huff_decode_at(const uint8_t *bits, uint64_t bit_phase, uint64_t bit_len, uint64_t count,
                                  const uint8_t *lengths, uint32_t cap, uint32_t maxlen, void *sym,
                                  int sym_bytes, lzb_dstatus *st, void *scratch, size_t scratch_bytes,
                                  void *stream) {
    if (bit_phase > 7) return LZB_E_ARG;
    return huff_decode_impl(bits, (uint32_t)bit_phase, bit_len, count, lengths, cap, maxlen, sym, sym_bytes,
                            st, scratch, scratch_bytes, stream);
}

// ---------------------------------------------------------------------------
// Bit-range decode: one rank of a multi-GPU decompression of ONE stream
// (SURVEY §8e).  Rank k owns the stream bits [bit_lo, bit_hi); bit_lo is a
// multiple of LZB_DEC_RANGE_ALIGN, so its subsequences are the whole-stream
// decoder's.  Pass 1 (lzb_huff_range_maps) composes the range's transfer map
// F_k(phase) = (symbols, exit phase); the host chains F_0..F_{k-1} from phase 0
// (one all-gather of maxlen words per rank) to get the range's entry phase
// and first symbol; pass 2 (lzb_huff_range_decode) resolves and decodes.
// ---------------------------------------------------------------------------
static int range_args(const uint8_t *bits, uint64_t bit_len, uint64_t bit_lo, uint64_t bit_hi,
                      const uint8_t *lengths, uint32_t cap, uint32_t maxlen, lzb_dstatus *st) {
    if (!bits || !lengths || !st || cap == 0 || maxlen == 0 || maxlen > 64) return LZB_E_ARG;
    if (bit_lo % LZB_DEC_RANGE_ALIGN != 0 || bit_lo >= bit_hi || bit_hi > bit_len) return LZB_E_ARG;
    if (bit_hi != bit_len && bit_hi % LZB_DEC_RANGE_ALIGN != 0) return LZB_E_ARG;
    if (reinterpret_cast<uintptr_t>(bits) & 3) return LZB_E_ARG;
    return LZB_OK;
}

extern "C" size_t lzb_huff_range_scratch_bytes(uint64_t range_bits, uint32_t maxlen, uint32_t cap) {
    return lzb_huff_decode_scratch_bytes(range_bits, maxlen, cap);
}

extern "C" int lzb_huff_range_maps(const uint8_t *bits, uint64_t bit_len, uint64_t bit_lo, uint64_t bit_hi,
                                   const uint8_t *lengths, uint32_t cap, uint32_t maxlen, uint64_t *fmap,
                                   lzb_dstatus *st, void *scratch, size_t scratch_bytes, void *stream) {
    int rc = range_args(bits, bit_len, bit_lo, bit_hi, lengths, cap, maxlen, st);
    if (rc != LZB_OK || !fmap) return rc != LZB_OK ? rc : LZB_E_ARG;
    cudaStream_t s = as_stream(stream);
    LZB_CUDA_TRY(cudaMemsetAsync(st, 0, sizeof(lzb_dstatus), s));
    DecParams p;
    DecLayout L;
    rc = dec_setup(bits + bit_lo / 8, 0, bit_hi - bit_lo, bit_len - bit_lo, 0, lengths, cap, maxlen, nullptr,
                   st, scratch, scratch_bytes, s, true, p, L);
    if (rc != LZB_OK) return rc;
    p.open_end = bit_hi < bit_len;
    if ((rc = dec_maps(p, L, s)) != LZB_OK) return rc;
    // the composition is always needed here (F_k for every entry phase)
    LZB_CUDA_TRY(cudaMemsetAsync(p.nonuni + 2, 1, sizeof(unsigned int), s));
    if ((rc = dec_compose(p, L, s, p.nonuni + 2)) != LZB_OK) return rc;
    k_dec_compose<uint64_t><<<(unsigned)((L.P + 63) / 64), 64, 0, s>>>(p.g2, L.ng2, L.P, (uint32_t)L.ng2,
                                                                     fmap, 1, p.nonuni + 2);
    LZB_LAUNCH_CHECK();
    return LZB_OK;
}

extern "C" int lzb_huff_range_decode(const uint8_t *bits, uint64_t bit_len, uint64_t bit_lo, uint64_t bit_hi,
                                     const uint8_t *lengths, uint32_t cap, uint32_t maxlen, uint32_t entry,
                                     uint32_t exit_phase, uint64_t count, void *sym, int sym_bytes,
                                     lzb_dstatus *st, void *scratch, size_t scratch_bytes, void *stream) {
    int rc = range_args(bits, bit_len, bit_lo, bit_hi, lengths, cap, maxlen, st);
    if (rc != LZB_OK) return rc;
    if ((sym_bytes != 2 && sym_bytes != 4) || entry >= maxlen) return LZB_E_ARG;
    const bool open = bit_hi < bit_len;
    if (open && exit_phase >= maxlen) return LZB_E_ARG;
    if (count == 0) return open ? LZB_E_ARG : LZB_OK;
    if (!sym) return LZB_E_ARG;
    cudaStream_t s = as_stream(stream);
    DecParams p;
    DecLayout L;
    rc = dec_setup(bits + bit_lo / 8, 0, bit_hi - bit_lo, bit_len - bit_lo, count, lengths, cap, maxlen, sym,
                   st, scratch, scratch_bytes, s, false, p, L);
    if (rc != LZB_OK) return rc;
    p.open_end = open;
    p.entry0 = entry;
    p.exit_expect = open ? exit_phase : kExitEnd;
    return dec_resolve_final(p, L, s, sym_bytes, cap);
}
