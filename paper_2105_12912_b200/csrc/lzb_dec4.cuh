// K5 v4: two passes over the dense Huffman bit stream, then a tile decoder
// that writes symbols straight into a consumer's shared-memory tile.
// Reference semantics: P/huffman.py:64-122 (one dense MSB-first stream, no
// offsets, canonical code book).
//
// Layout: the stream is cut into subsequences of 4096 bits (one warp each)
// and microblocks of 128 bits (one lane each).  A code word belongs to the
// microblock in which it STARTS.
//
// Pass M  k_dec4_count (warp per subsequence):
//   A) every lane decodes its microblock from the microblock start ("phase 0",
//      count-only boundary LUT: up to 12 code words per lookup), keeping the
//      code-word starts of the first 64 bits in a bitmap;
//   B) chain fixpoint inside the subsequence: lane i's entry is lane i-1's
//      exit; if that entry is a phase-0 start of lane i the counts follow
//      from a popcount, else lane i walks code words until it joins its
//      phase-0 path or reaches its end (then the walk IS the decode).
//   Lane 0 assumes entry 0.  Output per microblock (count << 8 | entry), per
//   subsequence lane 0's bitmap / phase-0 exit, the code words of lanes
//   1..31 and the chain's exit phase into the next subsequence.
// Pass S  k_dec4_resolve (thread per subsequence, single-pass look-back scan):
//   the true entry of subsequence s is the chain exit of s-1 (Huffman codes
//   self-synchronise: the chain exit does not depend on where lane 0 entered
//   once its path joins lane 0's phase-0 path).  Lane 0's count is corrected
//   from the bitmap or a short walk; a walk that leaves lane 0's microblock
//   at a different exit than phase 0 (a book that does not resynchronise in
//   128 bits), any invalid code word, a count mismatch or a missing END
//   raises LZB_E_RETRY: the caller then runs the exhaustive decoder
//   (lzb_huff_decode_robust, transfer maps over every entry phase), which
//   also adjudicates corrupt streams.  Outputs: every microblock's true entry
//   and count, every subsequence's first symbol offset.
// The final decode (k_dec_final9 in plan mode, lzb_dec3.cuh) then writes the
// symbols: warp per subsequence, lane per microblock from its planned entry.
//
// Measured and rejected (C5q, 512x2048^2 f32): fusing the final decode into
// K6 (tiles of chunks decoded straight into shared memory and reconstructed
// there, no code array in HBM) -- 6.5 ms for the fused kernel against 2.4 ms
// (final decode) + 2.9 ms (K6) separately: the fused CTA either idles its
// lanes on partially covered tiles or runs at 16-24 resident warps, and the
// thread-per-microblock decode chains are latency-bound at that occupancy.
#pragma once

#include "lzb_common.cuh"
#include "lzb_dectab.cuh"

namespace lzb {

constexpr uint32_t kFullMask = 0xffffffffu;
constexpr uint32_t kD4MB = 128;            // bits per microblock (lane)
constexpr uint32_t kD4S = 32 * kD4MB;      // bits per subsequence (warp)
constexpr uint8_t kD4Bad = 0xFF;
constexpr int kD4Warps = 8;                // k_dec4_count CTA
constexpr int kD4ResolveThreads = 256;     // k_dec4_resolve CTA (one subsequence per thread)

struct D4Plan {
    const uint32_t *words;  // 4-byte aligned base of the stream
    uint32_t head;          // bit offset of the first stream bit inside words[0]
    uint64_t nwords;
    uint64_t bit_len, count;
    uint64_t T;       // subsequences
    uint64_t nmb;     // microblocks holding stream bits
    const DecTables *tab;
    const uint32_t *syms;  // symbols in (length, symbol) order
    int32_t base8;         // lut8 byte deltas are relative to this symbol
    uint16_t *cp;     // per microblock (32 T): count << 8 | entry offset
    uint64_t *soff;   // per subsequence: stream index of its first code word's symbol
    uint64_t *sbm;    // per subsequence: lane 0 phase-0 starts in bits 0..63
    uint32_t *srest;  // per subsequence: code words of lanes 1..31 (chain)
    uint8_t *sx0;     // per subsequence: lane 0 phase-0 exit (kD4Bad: invalid)
    uint8_t *sexit;   // per subsequence: chain exit phase into the next one / kExitEnd / kD4Bad
    uint8_t *sirr;    // per subsequence: 1 = the true path joins the chain after microblock 0
    uint64_t *lb;     // look-back words, one per k_dec4_resolve tile
    unsigned int *ticket;
    lzb_dstatus *st;
};

// ---------------------------------------------------------------------------
// register bit window: 7 big-endian stream words (224 bits >= head 31 + 128 +
// a 64-bit code word), consumed from the front
// ---------------------------------------------------------------------------
struct D4Win {
    uint32_t w0, w1, w2, w3, w4, w5, w6;
    uint32_t sh;
    __device__ __forceinline__ void load(const D4Plan &p, uint64_t wi, uint32_t bit) {
        const uint32_t *s = p.words + wi;
        const uint64_t left = wi < p.nwords ? p.nwords - wi : 0;
        w0 = left > 0 ? bswap32(__ldg(s)) : 0u;
        w1 = left > 1 ? bswap32(__ldg(s + 1)) : 0u;
        w2 = left > 2 ? bswap32(__ldg(s + 2)) : 0u;
        w3 = left > 3 ? bswap32(__ldg(s + 3)) : 0u;
        w4 = left > 4 ? bswap32(__ldg(s + 4)) : 0u;
        w5 = left > 5 ? bswap32(__ldg(s + 5)) : 0u;
        w6 = left > 6 ? bswap32(__ldg(s + 6)) : 0u;
        sh = 0;
        adv64(bit);
    }
    __device__ __forceinline__ void shift() {
        w0 = w1;
        w1 = w2;
        w2 = w3;
        w3 = w4;
        w4 = w5;
        w5 = w6;
        w6 = 0;
    }
    __device__ __forceinline__ uint32_t peek12() const { return __funnelshift_l(w1, w0, sh) >> (32 - kLutBits); }
    __device__ __forceinline__ uint64_t peek64() const {
        return ((uint64_t)__funnelshift_l(w1, w0, sh) << 32) | __funnelshift_l(w2, w1, sh);
    }
    __device__ __forceinline__ void adv(uint32_t L) {  // L <= 32
        sh += L;
        if (sh >= 32) {
            sh -= 32;
            shift();
        }
    }
    __device__ __forceinline__ void adv64(uint32_t L) {  // L <= 95
        sh += L;
        while (sh >= 32) {
            sh -= 32;
            shift();
        }
    }
};

// microblock m's window, positioned at microblock bit `rel`
__device__ __forceinline__ void d4_window(const D4Plan &p, uint64_t m, uint32_t rel, D4Win &r) {
    const uint64_t a = (uint64_t)p.head + m * kD4MB;  // absolute word-stream bit
    r.load(p, a >> 5, (uint32_t)(a & 31) + rel);
}

// Streaming reader over the whole stream in global memory (pass S's rare
// full-subsequence walks): two or three word loads per peek, no state.
struct GRd {
    const D4Plan *p;
    uint64_t pos;  // absolute word-stream bit
    __device__ __forceinline__ uint32_t word(uint64_t w) const {
        return w < p->nwords ? bswap32(__ldg(p->words + w)) : 0u;
    }
    __device__ __forceinline__ uint32_t peek32() const {
        const uint64_t w = pos >> 5;
        return __funnelshift_l(word(w + 1), word(w), (uint32_t)(pos & 31));
    }
    __device__ __forceinline__ uint32_t peek12() const { return peek32() >> (32 - kLutBits); }
    __device__ __forceinline__ uint64_t peek64() const {
        const uint64_t w = pos >> 5;
        const uint32_t sh = (uint32_t)(pos & 31), w1 = word(w + 1);
        return ((uint64_t)__funnelshift_l(w1, word(w), sh) << 32) | __funnelshift_l(word(w + 2), w1, sh);
    }
    __device__ __forceinline__ void adv(uint32_t L) { pos += L; }
    __device__ __forceinline__ void adv64(uint32_t L) { pos += L; }
};

// ---------------------------------------------------------------------------
// shared-memory access through 32-bit shared addresses (no generic->shared
// conversion in the decode loops)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds8(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds16(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
// A shared address held in a register (the compiler may otherwise rebuild it
// from the CTA's shared window base inside hot loops).
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
    asm volatile("" : "+r"(a));
    return a;
}

// Bit reader over stream words staged in shared memory (memory byte order):
// w0:w1 hold the 64 bits at the position, sh < 32 the offset inside w0.
struct SRd {
    uint32_t a, w0, w1, sh;  // a: shared address of the word after w1
    __device__ __forceinline__ void init(uint32_t stg_s, uint32_t bit) {
        const uint32_t wa = stg_s + ((bit >> 5) << 2);
        sh = bit & 31;
        w0 = bswap32(lds32(wa));
        w1 = bswap32(lds32(wa + 4));
        a = wa + 8;
    }
    __device__ __forceinline__ uint32_t peek32() const { return __funnelshift_l(w1, w0, sh); }
    __device__ __forceinline__ uint32_t peek12() const { return peek32() >> (32 - kLutBits); }
    __device__ __forceinline__ uint64_t peek64() const {
        return ((uint64_t)peek32() << 32) | __funnelshift_l(bswap32(lds32(a)), w1, sh);
    }
    __device__ __forceinline__ void adv(uint32_t L) {  // L <= 32
        sh += L;
        if (sh >= 32) {
            sh -= 32;
            w0 = w1;
            w1 = bswap32(lds32(a));
            a += 4;
        }
    }
    __device__ __forceinline__ void adv64(uint32_t L) {  // L <= 64
        if (L > 32) {
            adv(32);
            L -= 32;
        }
        adv(L);
    }
};

// LUT access: shared-memory copies (pass M) or the global tables (pass S)
struct LutS {
    uint32_t b, c, l1;  // shared addresses of lutb, lutc, lut1
    const DecCanon *can;
    __device__ __forceinline__ uint32_t lb(uint32_t pk) const { return lds32(b + 4 * pk); }
    __device__ __forceinline__ uint32_t lc(uint32_t pk) const { return lds32(c + 4 * pk); }
    __device__ __forceinline__ uint32_t ll1(uint32_t pk) const { return lds8(l1 + pk); }
};
struct LutG {
    const DecTables *t;
    const DecCanon *can;
    __device__ __forceinline__ uint32_t lb(uint32_t pk) const { return __ldg(&t->lutb[pk]); }
    __device__ __forceinline__ uint32_t lc(uint32_t pk) const { return __ldg(&t->lutc[pk]); }
    __device__ __forceinline__ uint32_t ll1(uint32_t pk) const { return __ldg(&t->lut1[pk]); }
};

// length of a code word longer than the LUT (canonical tables from L0)
__device__ __forceinline__ uint32_t d4_len_long(const DecCanon *tab, uint64_t v, uint32_t L0) {
    for (uint32_t L = L0; L <= tab->maxlen; L++) {
        const uint64_t c = v >> (64 - L);
        if (c >= tab->first[L] && c - tab->first[L] < tab->cnt[L]) return L;
    }
    return 0;
}
__device__ __forceinline__ uint32_t d4_sym_long(const DecCanon *tab, const uint32_t *syms, uint64_t v,
                                                uint32_t L0, uint32_t &sym) {
    for (uint32_t L = L0; L <= tab->maxlen; L++) {
        const uint64_t c = v >> (64 - L);
        const uint64_t f = tab->first[L];
        if (c >= f && c - f < tab->cnt[L]) {
            sym = syms[tab->off[L] + (uint32_t)(c - f)];
            return L;
        }
    }
    return 0;
}
// length of the code word at the reader (0: invalid prefix)
template <typename Rd, typename Lut>
__device__ __forceinline__ uint32_t d4_len(const Lut &lt, const Rd &r) {
    const uint32_t l1 = lt.ll1(r.peek12());
    if (l1 & 0x80u) return d4_len_long(lt.can, r.peek64(), l1 & 0x7Fu);
    return l1;
}

// Count-only decode of the code words STARTING in [rel, stop), reader at rel;
// code words must end by endrel (END).  REC: phase-0 starts below bit 64 go
// to bm.  false: invalid prefix or a code word past END.
template <bool REC, typename Rd, typename Lut>
__device__ __forceinline__ bool d4_count(Rd &r, const Lut &lt, uint32_t &rel, uint32_t stop, uint32_t endrel,
                                         uint32_t &cnt, uint64_t &bm) {
    // one loop for every case, so the lanes of a warp stay converged
    while (rel < stop) {
        const uint32_t pk = r.peek12();
        const uint32_t e = lt.lb(pk);
        uint32_t n = e & 15u, used = (e >> 4) & 15u, starts = e >> 8;
        if (n == 0) {  // a code word longer than the LUT (or an invalid prefix)
            const uint32_t L = d4_len(lt, r);
            if (L == 0 || rel + L > endrel) return false;
            if (REC && rel < 64) bm |= 1ull << rel;
            cnt++;
            rel += L;
            r.adv64(L);
            continue;
        }
        if (stop - rel < (uint32_t)kLutBits) {  // drop code words starting at or after stop
            const uint32_t hi = starts & (0xFFFu << (stop - rel));
            n -= __popc(hi);
            used = hi ? (uint32_t)(__ffs(hi) - 1) : used;
            starts &= ~hi;
            if (rel + used > endrel) return false;
        }
        if (REC && rel < 64) bm |= (uint64_t)starts << rel;
        cnt += n;
        rel += used;
        r.adv(used);
    }
    return true;
}

// Walk code words from pos (reader at pos) until a start recorded in bm
// (phase-0 start below bit 64; returns 1, pos = that start) or the first
// start at / after stop (returns 0, pos = exit); 2 = invalid / past END.
// cnt += code words walked before the returned position.
template <typename Rd, typename Lut>
__device__ __forceinline__ int d4_walk(Rd &r, const Lut &lt, uint32_t &pos, uint32_t stop, uint32_t endrel,
                                       uint64_t bm, uint32_t &cnt) {
    if (pos >= stop) return 0;
    if (pos < 64 && ((bm >> pos) & 1ull)) return 1;
    while (true) {
        const uint32_t e = lt.lb(r.peek12());
        const uint32_t n = e & 15u, used = (e >> 4) & 15u;
        if (n == 0 || pos + (uint32_t)kLutBits > stop) {  // one code word at a time
            const uint32_t L = d4_len(lt, r);
            if (L == 0 || pos + L > endrel) return 2;
            pos += L;
            cnt++;
            if (pos >= stop) return 0;
            if (pos < 64 && ((bm >> pos) & 1ull)) return 1;
            r.adv64(L);
            continue;
        }
        // code-word boundaries at pos + j, j = 1..used  <->  bit j-1 of ends
        const uint32_t ends = ((e >> 8) >> 1) | (1u << (used - 1));
        const uint32_t hit = pos < 63 ? ends & (uint32_t)(bm >> (pos + 1)) : 0u;
        if (hit) {
            const uint32_t j = __ffs(hit);
            cnt += __popc(ends & ((1u << j) - 1u));
            pos += j;
            return 1;
        }
        pos += used;
        cnt += n;
        if (pos >= stop) return 0;
        r.adv(used);
    }
}

__device__ __forceinline__ uint32_t d4_rank64(uint64_t bm, uint32_t q) {  // set bits below q (< 64)
    return __popcll(bm & ((1ull << q) - 1ull));
}

// Asynchronous copy of stream words [wlo, wlo + nw) into shared memory at
// dst_s (4-byte pieces, zero past the stream), by threads tid = 0..nthr-1.
__device__ __forceinline__ void d4_stage_words(const D4Plan &p, uint64_t wlo, uint32_t nw, uint32_t dst_s,
                                               uint32_t tid, uint32_t nthr) {
    if ((((reinterpret_cast<uintptr_t>(p.words + wlo)) | dst_s) & 15) == 0 && wlo + ((nw + 3) & ~3u) <= p.nwords) {
        for (uint32_t i = tid; 4 * i < nw; i += nthr)  // 16-byte pieces
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst_s + 16 * i), "l"(p.words + wlo + 4 * i)
                         : "memory");
        return;
    }
    for (uint32_t i = tid; i < nw; i += nthr) {
        const uint64_t w = wlo + i;
        const bool in = w < p.nwords;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst_s + 4 * i),
                     "l"(p.words + (in ? w : 0)), "r"(in ? 4 : 0)
                     : "memory");
    }
}

// Host side (lzb_huff.cu): tables, LUTs, pass M and pass S on stream `bits`
// (first bit at bit `bit_phase` of bits[0]).  Scratch carve-up shared with the
// consumers; LZB_E_RETRY lands in st when the plan is unusable.
size_t d4_scratch_bytes(uint64_t bit_len, uint64_t count, uint32_t cap);
int d4_plan(const uint8_t *bits, uint32_t bit_phase, uint64_t bit_len, uint64_t count,
            const uint8_t *lengths, uint32_t cap, uint32_t maxlen, lzb_dstatus *st, Scratch &sc,
            cudaStream_t s, D4Plan &p);

static_assert(offsetof(DecTables, cnt) - offsetof(DecTables, first) == offsetof(DecCanon, cnt) &&
                  offsetof(DecTables, off) - offsetof(DecTables, first) == offsetof(DecCanon, off) &&
                  offsetof(DecTables, maxlen) - offsetof(DecTables, first) == offsetof(DecCanon, maxlen),
              "DecCanon must mirror DecTables' canonical fields");

#ifdef LZB_DEC4_KERNELS
constexpr uint32_t kD4StgW = 136;  // staged words per subsequence: 128 + head + a 64-bit code word + peek

// cp.async the words of subsequence t into a warp's stage (zero past the stream)
__device__ __forceinline__ void d4_stage_sub(const D4Plan &p, uint64_t t, uint32_t dst_s, uint32_t lane) {
    if (t < p.T) d4_stage_words(p, t * 128, kD4StgW, dst_s, lane, 32);
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// ---------------------------------------------------------------------------
// Pass M
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kD4Warps * 32) k_dec4_count(D4Plan p) {
    __shared__ uint32_t s_b[kLutSize];
    __shared__ uint8_t s_l1[kLutSize];
    __shared__ DecCanon s_can;
    __shared__ __align__(16) uint32_t s_w[kD4Warps][2][kD4StgW];
    for (uint32_t i = threadIdx.x; i < kLutSize; i += blockDim.x) {
        s_b[i] = p.tab->lutb[i];
        s_l1[i] = p.tab->lut1[i];
    }
    load_canon(s_can, p.tab);
    __syncthreads();
    if (p.st->code) return;  // invalid code book (k_dec_tables)
    const LutS lt{smem_addr(s_b), 0u, smem_addr(s_l1), &s_can};
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    const uint32_t w_s = smem_addr(&s_w[warp][0][0]);
    const uint64_t nwt = (uint64_t)gridDim.x * kD4Warps;
    uint64_t t = (uint64_t)blockIdx.x * kD4Warps + warp;
    uint32_t sb = 0;
    d4_stage_sub(p, t, w_s, lane);
    for (; t < p.T; t += nwt, sb ^= 1) {
        d4_stage_sub(p, t + nwt, w_s + (sb ^ 1) * kD4StgW * 4, lane);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncwarp();
        const uint32_t stg = w_s + sb * kD4StgW * 4;
        const uint64_t m = t * 32 + lane;
        const uint64_t b0 = m * kD4MB;
        const bool act = b0 < p.bit_len;
        const uint32_t stop = act ? (uint32_t)umin64(kD4MB, p.bit_len - b0) : 0u;
        const uint32_t endrel = act ? (uint32_t)umin64(p.bit_len - b0, 0xFFFFFF00u) : 0u;
        const uint32_t lbit = lane * kD4MB + p.head;  // the lane's microblock in the stage
        // ---- A: phase-0 decode ----
        uint32_t x0 = 0, c0 = 0;
        uint64_t bm = 0;
        bool ok0 = true;
        if (act) {
            SRd r;
            r.init(stg, lbit);
            ok0 = d4_count<true>(r, lt, x0, stop, endrel, c0, bm);
        }
        // ---- B: chain fixpoint (lane 0 enters at 0) ----
        uint32_t x = x0, cnt = c0, ent = 0;
        bool val = ok0;
        bool need = act && lane > 0;
        while (__any_sync(kFullMask, need)) {
            const uint32_t px = __shfl_up_sync(kFullMask, x, 1);
            const bool pv = __shfl_up_sync(kFullMask, val, 1);
            bool changed = false;
            if (need) {
                uint32_t pos = px - kD4MB, k = 0, nx, nc;
                bool lk;
                SRd r;
                r.init(stg, lbit + pos);
                const int w = d4_walk(r, lt, pos, stop, endrel, bm, k);
                if (w == 2) {
                    lk = false;
                    nx = pos;
                    nc = k;
                } else if (w == 1) {
                    lk = ok0;
                    nc = k + c0 - d4_rank64(bm, pos);
                    nx = x0;
                } else {
                    lk = true;
                    nc = k;
                    nx = pos;
                }
                const bool v = pv && lk;
                changed = (nx != x) || (v != val);
                ent = px - kD4MB;
                x = nx;
                cnt = nc;
                val = v;
            }
            need = __shfl_up_sync(kFullMask, changed, 1) && act && lane > 0;
        }
        p.cp[m] = act ? (uint16_t)((cnt << 8) | ent) : (uint16_t)0;
        const uint32_t rest = __reduce_add_sync(kFullMask, (act && lane > 0) ? cnt : 0u);
        const uint32_t la = (uint32_t)umin64(31, (p.bit_len - 1 - t * kD4S) / kD4MB);  // last active lane
        const uint32_t xl = __shfl_sync(kFullMask, x, la);
        const uint32_t stl = __shfl_sync(kFullMask, stop, la);
        const bool allv = __all_sync(kFullMask, !act || val);
        if (lane == 0) {
            p.sbm[t] = bm;
            p.sx0[t] = ok0 ? (uint8_t)x0 : kD4Bad;
            p.srest[t] = rest;
            uint8_t ex;
            if (!allv) ex = kD4Bad;
            else if (t == p.T - 1) ex = xl == stl ? kExitEnd : kD4Bad;
            else ex = (uint8_t)(xl - kD4MB);
            p.sexit[t] = ex;
        }
        __syncwarp();  // every lane is done with this stage buffer
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
}

// ---------------------------------------------------------------------------
// Pass S
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kD4ResolveThreads) k_dec4_resolve(D4Plan p) {
    __shared__ uint64_t s_scan[33];
    __shared__ uint64_t s_tile, s_ex;
    __shared__ int s_retry;
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    const uint64_t ntl = (p.T + kD4ResolveThreads - 1) / kD4ResolveThreads;
    // DecTables' canonical fields have DecCanon's layout (static_assert above)
    const LutG lt{p.tab, reinterpret_cast<const DecCanon *>(&p.tab->first[0])};
    while (true) {
        if (threadIdx.x == 0) {
            s_tile = atomicAdd(p.ticket, 1u);
            s_retry = 0;
        }
        __syncthreads();
        const uint64_t tl = s_tile;
        if (tl >= ntl) break;
        const uint64_t s = tl * kD4ResolveThreads + threadIdx.x;
        uint64_t total = 0;
        uint32_t cnt0 = 0, e = 0;
        bool retry = p.st->code != 0, irregular = false;
        if (s < p.T) {
            const uint32_t ev = s == 0 ? 0u : p.sexit[s - 1];
            const uint32_t x0 = p.sx0[s];
            const uint64_t m = s * 32;
            const uint64_t b0 = m * kD4MB;
            const uint32_t stop = (uint32_t)umin64(kD4MB, p.bit_len - b0);
            const uint32_t c0 = p.cp[m] >> 8;
            const uint64_t bm = p.sbm[s];
            if (ev >= 64 || x0 == kD4Bad || ev >= stop) {
                retry = true;
            } else {
                e = ev;
                if ((bm >> e) & 1ull) {
                    cnt0 = c0 - d4_rank64(bm, e);
                } else {
                    D4Win r;
                    d4_window(p, m, e, r);
                    uint32_t pos = e, k = 0;
                    const uint32_t endrel = (uint32_t)umin64(p.bit_len - b0, 0xFFFFFF00u);
                    const int w = d4_walk(r, lt, pos, stop, endrel, bm, k);
                    if (w == 1) cnt0 = k + c0 - d4_rank64(bm, pos);
                    else if (w == 0 && pos == x0) cnt0 = k;
                    else if (w == 2) retry = true;
                    else irregular = true;
                }
            }
            if (irregular) {
                // the true path has not joined the chain by the end of
                // microblock 0: walk on microblock by microblock until it
                // enters one at the chain's entry (pass M's cp[]); from there
                // on the counts are the chain's.  Otherwise (rare) the walk
                // covers the whole subsequence and its exit must agree with
                // pass M's.  The final decode re-resolves the entries.
                const uint32_t sbits = (uint32_t)umin64(kD4S, p.bit_len - b0);
                const uint32_t endrel = (uint32_t)umin64(p.bit_len - b0, 0xFFFFFF00u);
                GRd g{&p, (uint64_t)p.head + b0 + e};
                uint32_t rel = e, c = 0, rest = p.srest[s];
                uint64_t dummy = 0;
                bool joined = false;
                for (uint32_t j = 0; j < 32 && rel < sbits && !retry; j++) {
                    const uint32_t mb_end = (j + 1) * kD4MB < sbits ? (j + 1) * kD4MB : sbits;
                    if (!d4_count<false>(g, lt, rel, mb_end, endrel, c, dummy)) retry = true;
                    if (retry || j == 31 || mb_end == sbits) break;
                    const uint32_t cj = p.cp[m + j + 1];
                    if (rel == mb_end + (cj & 0xFFu)) {  // on the chain from here
                        c += rest;
                        joined = true;
                        break;
                    }
                    rest -= cj >> 8;
                }
                if (!joined) {
                    const bool lastsub = s == p.T - 1;
                    if (lastsub ? rel != sbits : rel - kD4S != (uint32_t)p.sexit[s]) retry = true;  // exit must agree
                }
                total = c;
                cnt0 = c0;
                p.sirr[s] = 1;
            } else {
                total = (uint64_t)cnt0 + p.srest[s];
                if (s == p.T - 1 && p.sexit[s] != kExitEnd) retry = true;
                p.sirr[s] = 0;
            }
        }
        uint64_t tot;
        const uint64_t off = block_exclusive_scan<uint64_t>(total, s_scan, &tot);
        if (warp == 0) {
            const uint64_t ex = lookback_warp(p.lb, tl, tot);
            if (lane == 0) s_ex = ex;
        }
        if (retry) s_retry = 1;
        __syncthreads();
        const uint64_t soff = s_ex + off;
        if (s < p.T) {
            p.cp[s * 32] = (uint16_t)((cnt0 << 8) | e);
            if (s == p.T - 1 && soff + total != p.count) s_retry = 1;
        }
        __syncthreads();
        if (s_retry && threadIdx.x == 0) set_status(p.st, LZB_E_RETRY);
        if (s < p.T) p.soff[s] = soff;
        __syncthreads();
    }
}

#endif  // LZB_DEC4_KERNELS

}  // namespace lzb
