// K5 v3: warp per subsequence, lane per 128-bit microblock.  Included by
// lzb_huff.cu (inside namespace lzb) after the shared decode pieces
// (DecParams, DecCanon, the LUTs).  Reference: P/huffman.py:64-122 (canonical
// decode of one dense MSB-first stream; the archive has no offsets).
//
// The stream is cut into subsequences of kS3 = 4096 bits (one warp each),
// and each subsequence into 32 microblocks of kMB = 128 bits (one lane each).
// A warp stages its subsequence's 512 stream bytes (+ a tail) in shared
// memory with one coalesced cp.async pass, double-buffered across the warp's
// subsequences, and every lane reads its bits from there.
//
// k_dec_maps3 (per subsequence):
//   A) every lane decodes its microblock from the microblock start ("phase
//      0"; boundary LUT, up to 12 code words per lookup), recording the
//      code-word starts in a 128-bit bitmap, its count and its exit;
//   B) chain fixpoint: the true path of the subsequence's phase 0 enters
//      microblock i where microblock i-1's path exits.  A lane whose entry is
//      a recorded start of its own phase-0 path is resolved by a popcount;
//      otherwise it walks single code words until it hits one (Huffman codes
//      self-synchronise within a few code words) or leaves its microblock.
//      Lanes re-resolve while their predecessor's exit changes (<= 31 rounds,
//      1 in practice);
//   C) entry phases 1..P-1 of the subsequence walk microblock by microblock
//      until they join the chain; phases that have not joined it by the end
//      of microblock 0 are marked irregular for the final pass.
//   Output: the transfer map of every entry phase (composed by the
//   hierarchical passes into each subsequence's true entry and symbol
//   offset), and per microblock the chain's entry offset and code-word count.
// k_dec_final9 (per subsequence, u16 symbols): every lane decodes its
//   microblock from its chain entry (lane 0 from the subsequence's true
//   entry) with the byte LUT into a per-warp stage laid out like the output
//   range, then the warp widens and copies the stage out with coalesced
//   16-byte stores.  Irregular entries first re-resolve the lanes' starts
//   and counts by a count-only fixpoint.
#pragma once
// (included inside namespace lzb)

constexpr uint32_t kD3Full = 0xffffffffu;
constexpr uint32_t kMB = 128;       // bits per lane (microblock)
constexpr uint32_t kS3 = 32 * kMB;  // bits per subsequence (warp)
constexpr uint32_t kStgWords = 136; // staged stream words per subsequence (128 + tail)
constexpr int kD3Warps = 8;         // k_dec_maps3 CTA

__device__ __forceinline__ bool bm2_test(uint64_t b0, uint64_t b1, uint32_t q) {  // q < 128
    const uint64_t w = q < 64 ? b0 : b1;
    return ((w >> (q & 63)) & 1ull) != 0;
}
__device__ __forceinline__ uint32_t bm2_rank(uint64_t b0, uint64_t b1, uint32_t q) {  // set bits < q
    if (q <= 64) return q == 64 ? __popcll(b0) : __popcll(b0 & ((1ull << q) - 1ull));
    return __popcll(b0) + __popcll(b1 & ((1ull << (q - 64)) - 1ull));
}

// cp.async the stream words of subsequence t (global words 128 t ...) into
// a warp's stage; words past the stream are zero-filled.
__device__ __forceinline__ void d3_stage(const DecParams &p, uint64_t t, uint32_t s_addr, uint32_t lane) {
    if (t < p.T) {
        const uint64_t w0 = t * 128;
        if ((reinterpret_cast<uintptr_t>(p.words) & 15) == 0 && w0 + kStgWords <= p.nwords) {
            // 34 aligned 16-byte pieces
            for (uint32_t j = lane; j < kStgWords / 4; j += 32)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s_addr + 16 * j),
                             "l"(p.words + w0 + 4 * j)
                             : "memory");
        } else {
            for (uint32_t j = lane; j < kStgWords; j += 32) {
                const uint64_t w = w0 + j;
                const bool in = w < p.nwords;
                const uint32_t *src = p.words + (in ? w : 0);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(s_addr + 4 * j), "l"(src),
                             "r"(in ? 4 : 0)
                             : "memory");
            }
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void d3_stage_wait() {
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp();
}

// Bit window over a staged subsequence (raw big-endian stream words), read
// through 32-bit shared addresses (lds32): a generic pointer made the
// compiler rebuild the shared window base (S2UR + ULEA) at every refill.
struct SWin {
    uint32_t base;       // shared address of the stage
    uint32_t ad;         // shared address of the word after w2
    uint32_t sh;         // bit offset inside w0
    uint32_t w0, w1, w2;
    __device__ __forceinline__ void init(const uint32_t *st, uint32_t a) { init_s(smem_addr(st), a); }
    __device__ __forceinline__ void init_s(uint32_t b, uint32_t a) {  // a: stage bit
        base = b;
        const uint32_t wa = b + ((a >> 5) << 2);
        sh = a & 31;
        w0 = bswap32(lds32(wa));
        w1 = bswap32(lds32(wa + 4));
        w2 = bswap32(lds32(wa + 8));
        ad = wa + 12;
    }
    __device__ __forceinline__ uint32_t peek12() const { return __funnelshift_l(w1, w0, sh) >> (32 - kLutBits); }
    __device__ __forceinline__ uint64_t peek64() const {
        return ((uint64_t)__funnelshift_l(w1, w0, sh) << 32) | __funnelshift_l(w2, w1, sh);
    }
    __device__ __forceinline__ void consume(uint32_t L) {  // L <= 32
        sh += L;
        if (sh >= 32) {
            sh -= 32;
            w0 = w1;
            w1 = w2;
            w2 = bswap32(lds32(ad));
            ad += 4;
        }
    }
    __device__ __forceinline__ void skip(uint32_t L) {  // any L <= 64
        if (L <= 32) consume(L);
        else init_s(base, (ad - 12 - base) * 8 + sh + L);
    }
};

// Code word longer than 12 bits: canonical tables from the shortest length
// with this prefix (lut1 & 0x7F).  Returns the length, 0 if none matches.
__device__ __forceinline__ uint32_t dlen_long(const DecCanon *tab, uint64_t v, uint32_t L0) {
    for (uint32_t L = L0; L <= tab->maxlen; L++) {
        const uint64_t c = v >> (64 - L);
        const uint64_t f = tab->first[L], k = tab->cnt[L];
        if (c >= f && c - f < k) return L;
    }
    return 0;
}
__device__ __forceinline__ uint32_t dsym_long(const DecCanon *tab, const uint32_t *syms, uint64_t v,
                                              uint32_t L0, uint32_t &sym) {
    for (uint32_t L = L0; L <= tab->maxlen; L++) {
        const uint64_t c = v >> (64 - L);
        const uint64_t f = tab->first[L], k = tab->cnt[L];
        if (c >= f && c - f < k) {
            sym = syms[tab->off[L] + (uint32_t)(c - f)];
            return L;
        }
    }
    return 0;
}
// length of the code word at the window (0 = invalid)
__device__ __forceinline__ uint32_t d3_len(const uint8_t *s_l1, const DecCanon *tab, const SWin &r) {
    const uint32_t l1 = s_l1[r.peek12()];
    if (l1 & 0x80u) return dlen_long(tab, r.peek64(), l1 & 0x7Fu);
    return l1;
}

// Bulk decode (boundary LUT) of the code words STARTING in [rel, mstop);
// records their starts relative to b in (bm0, bm1) when REC.  Returns false on
// an invalid code word or one running past the stream end (endrel).
template <bool REC>
__device__ __forceinline__ bool d3_bulk(const uint32_t *stg, uint32_t head, const uint32_t *s_b,
                                        const uint8_t *s_l1, const DecCanon *tab, uint32_t b,
                                        uint32_t mstop, uint32_t endrel, uint32_t &rel, uint32_t &cnt,
                                        uint64_t &bm0, uint64_t &bm1) {
    if (rel >= mstop) return true;
    SWin r;
    r.init(stg, rel + head);
    while (rel < mstop) {
        const uint32_t pk = r.peek12();
        const uint32_t e = s_b[pk];
        uint32_t n = e & 15u, used = (e >> 4) & 15u, starts = e >> 8;
        if (n == 0) {  // first code word longer than the LUT, or an invalid prefix
            const uint32_t l1 = s_l1[pk];
            const uint32_t L = (l1 & 0x80u) ? dlen_long(tab, r.peek64(), l1 & 0x7Fu) : 0u;
            if (L == 0 || rel + L > endrel) return false;
            n = 1;
            used = L;
            starts = 1;
        } else {
            const uint32_t d = mstop - rel;
            if (d < (uint32_t)kLutBits) {  // drop code words starting at or after mstop
                const uint32_t hi = starts & (0xFFFu << d);
                n -= __popc(hi);
                used = hi ? (uint32_t)(__ffs(hi) - 1) : used;
                starts &= ~hi;
                if (rel + used > endrel) return false;
            }
        }
        if (REC) {
            const uint32_t q = rel - b;
            if (q < 64) {
                bm0 |= (uint64_t)starts << q;
                if (q > 52) bm1 |= (uint64_t)starts >> (64 - q);
            } else {
                bm1 |= (uint64_t)starts << (q - 64);
            }
        }
        cnt += n;
        rel += used;
        r.skip(used);
    }
    return true;
}

// bits q .. q+31 of the 128-bit start map (zero past bit 127)
__device__ __forceinline__ uint32_t bm2_win(uint64_t b0, uint64_t b1, uint32_t q) {
    uint64_t v;
    if (q < 64) v = (b0 >> q) | (q ? (b1 << (64 - q)) : 0ull);
    else if (q < 128) v = b1 >> (q - 64);
    else v = 0;
    return (uint32_t)v;
}

// Walk code words from pos until a code-word boundary is at / after mstop
// (returns 0) or is a start recorded in (bm0, bm1) relative to b (returns
// 1), or an invalid / truncated code word (returns 2); cnt counts the code
// words walked.  Up to 12 code words per boundary-LUT lookup; single code
// words for code words longer than the LUT and near the stream end.
__device__ __forceinline__ int d3_walk_lut(const uint32_t *stg, uint32_t head, const uint32_t *s_b,
                                           const uint8_t *s_l1, const DecCanon *tab, uint32_t &pos,
                                           uint32_t b, uint32_t mstop, uint32_t endrel, uint64_t bm0,
                                           uint64_t bm1, uint32_t &cnt) {
    if (pos >= mstop) return 0;
    if (bm2_test(bm0, bm1, pos - b)) return 1;
    SWin r;
    r.init(stg, pos + head);
    while (true) {
        const uint32_t e = s_b[r.peek12()];
        const uint32_t n = e & 15u, used = (e >> 4) & 15u;
        if (n == 0 || pos + (uint32_t)kLutBits > endrel) {
            const uint32_t L = d3_len(s_l1, tab, r);
            if (L == 0 || pos + L > endrel) return 2;
            pos += L;
            cnt++;
            if (pos >= mstop) return 0;
            if (bm2_test(bm0, bm1, pos - b)) return 1;
            r.skip(L);
            continue;
        }
        // boundary at pos + j  <->  bit j - 1 (1 <= j <= used)
        const uint32_t ends = ((e >> 8) >> 1) | (1u << (used - 1));
        uint32_t hit = ends & bm2_win(bm0, bm1, pos + 1 - b);
        const uint32_t dm = mstop - pos;  // >= 1
        if (dm <= used) hit |= ends & ~((1u << (dm - 1)) - 1u);
        if (hit) {
            const uint32_t j = __ffs(hit);
            cnt += __popc(ends & ((1u << j) - 1u));
            pos += j;
            return pos >= mstop ? 0 : 1;
        }
        pos += used;
        cnt += n;
        r.skip(used);
    }
}

// per-microblock data shared by the lanes of a warp in phase C
struct MbInfo {
    uint64_t bm0, bm1;  // phase-0 code-word starts (offsets from the microblock start)
    uint16_t x0;        // phase-0 exit (relative to the subsequence start)
    uint16_t c0;        // phase-0 code words
    uint16_t ent;       // chain entry
    uint16_t sin;       // chain code words in this and all later microblocks
    uint8_t ok0;        // phase-0 decode valid
    uint8_t vin;        // chain valid from this microblock on
    uint8_t pad[6];
};

__global__ void __launch_bounds__(kD3Warps * 32) k_dec_maps3(DecParams p) {
    __shared__ uint32_t s_b[kLutSize];
    __shared__ uint8_t s_l1[kLutSize];
    __shared__ DecCanon s_can;
    __shared__ MbInfo s_mb[kD3Warps][32];
    __shared__ __align__(16) uint32_t s_str[kD3Warps][2][kStgWords];
    for (uint32_t i = threadIdx.x; i < kLutSize; i += blockDim.x) {
        s_b[i] = p.tab->lutb[i];
        s_l1[i] = p.tab->lut1[i];
    }
    load_canon(s_can, p.tab);
    __syncthreads();
    const DecCanon *tab = &s_can;
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    MbInfo *mb = s_mb[warp];
    const uint32_t str_s = (uint32_t)__cvta_generic_to_shared(&s_str[warp][0][0]);
    const uint64_t nw = (uint64_t)gridDim.x * kD3Warps;
    uint64_t t = (uint64_t)blockIdx.x * kD3Warps + warp;
    uint32_t sb = 0;
    d3_stage(p, t, str_s, lane);
    for (; t < p.T; t += nw, sb ^= 1) {
        d3_stage(p, t + nw, str_s + (sb ^ 1) * kStgWords * 4, lane);
        d3_stage_wait();
        const uint32_t *stg = s_str[warp][sb];
        const uint64_t t0 = t * kS3;
        const bool last = t == p.T - 1 && !p.open_end;  // END semantics
        const uint32_t stop = last ? (uint32_t)(p.bit_len - t0) : kS3;
        const uint32_t endrel = (uint32_t)umin64(p.total_bits - t0, 0xFFFFFFF0u);
        const uint32_t la = (stop + kMB - 1) / kMB - 1;  // last active lane
        const uint32_t b = lane * kMB;
        const bool act = lane <= la;
        const uint32_t mstop = act ? min(b + kMB, stop) : b;

        // ---- A: phase-0 decode of every microblock ----
        uint32_t x0 = b, c0 = 0;
        uint64_t bm0 = 0, bm1 = 0;
        bool ok0 = true;
        if (act) ok0 = d3_bulk<true>(stg, p.head, s_b, s_l1, tab, b, mstop, endrel, x0, c0, bm0, bm1);

        // ---- B: chain fixpoint ----
        uint32_t x = x0, cnt = c0, ent = b;
        bool lok = ok0;  // this lane's resolution is a valid decode from ent
        bool val = ok0;  // ... and so is the whole chain up to here
        bool need = act && lane > 0;
        while (__any_sync(kD3Full, need)) {
            const uint32_t px = __shfl_up_sync(kD3Full, x, 1);
            const bool pv = __shfl_up_sync(kD3Full, val, 1);
            bool changed = false;
            if (need) {
                uint32_t pos = px, k = 0, nx, nc;
                bool lk;
                const int w = d3_walk_lut(stg, p.head, s_b, s_l1, tab, pos, b, mstop, endrel, bm0, bm1, k);
                if (w == 2) {
                    lk = false;
                    nx = pos;
                    nc = k;
                } else if (w == 1) {
                    lk = ok0;
                    nc = k + c0 - bm2_rank(bm0, bm1, pos - b);
                    nx = x0;
                } else {
                    lk = true;
                    nc = k;
                    nx = pos;
                }
                const bool v = pv && lk;
                changed = (nx != x) || (v != val);
                ent = px;
                x = nx;
                cnt = nc;
                lok = lk;
                val = v;
            }
            need = __shfl_up_sync(kD3Full, changed, 1) && act && lane > 0;
        }
        const uint32_t c_act = act ? cnt : 0u;
        // inclusive suffix sums of the counts (lanes >= this one)
        uint32_t sin = c_act;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_down_sync(kD3Full, sin, o);
            if (lane + o < 32) sin += v;
        }
        const uint32_t tot = __shfl_sync(kD3Full, sin, 0);
        const uint32_t badm = __ballot_sync(kD3Full, act && !lok);
        const bool vin = (badm >> lane) == 0;
        const uint32_t xl = __shfl_sync(kD3Full, x, la);
        const bool vl = __shfl_sync(kD3Full, val, la);
        uint32_t xraw;  // exit code of the chain from any valid join point
        if (last) xraw = (xl == stop) ? kExitEnd : kExitInvalid;
        else xraw = xl - stop;
        {
            MbInfo m;
            m.bm0 = bm0;
            m.bm1 = bm1;
            m.x0 = (uint16_t)x0;
            m.c0 = (uint16_t)c0;
            m.ent = (uint16_t)ent;
            m.sin = (uint16_t)sin;
            m.ok0 = ok0;
            m.vin = vin;
            mb[lane] = m;
        }
        p.cp[t * 32 + lane] = act ? (uint16_t)((cnt << 8) | ((ent - b) & 0xFFu)) : (uint16_t)0;
        __syncwarp();

        // ---- C: entry phases 1..P-1 ----
        uint64_t irr = 0;
        uint32_t emin = kExitInvalid, emax = 0;  // range of this lane's valid exit codes
        for (uint32_t ph = 1 + lane; ph < p.P; ph += 32) {
            uint32_t out = kExitInvalid;
            bool regular = false;
            if (ph <= stop && t0 + ph <= p.bit_len) {
                uint32_t pos = ph, c = 0;
                for (uint32_t k = 0;; k++) {
                    if (k > la) {  // past the subsequence end
                        uint32_t ex;
                        if (last) ex = (pos == stop) ? kExitEnd : kExitInvalid;
                        else ex = pos - stop;
                        out = ex == kExitInvalid ? kExitInvalid : ((c << 8) | ex);
                        if (k == 1) regular = true;
                        break;
                    }
                    const MbInfo &m = mb[k];
                    if (k > 0 && pos == m.ent && m.vin) {  // joined the chain
                        out = xraw == kExitInvalid ? kExitInvalid : (((c + m.sin) << 8) | xraw);
                        if (k == 1) regular = true;
                        break;
                    }
                    const uint32_t bk = k * kMB, ms = min(bk + kMB, stop);
                    const int w = d3_walk_lut(stg, p.head, s_b, s_l1, tab, pos, bk, ms, endrel, m.bm0, m.bm1, c);
                    if (w == 2) break;
                    if (w == 1) {  // joined microblock k's phase-0 path
                        if (!m.ok0) break;
                        c += m.c0 - bm2_rank(m.bm0, m.bm1, pos - bk);
                        pos = m.x0;
                    }
                }
            }
            if (!regular) irr |= 1ull << ph;
            if (out != kExitInvalid) {
                emin = min(emin, out & 0xFFu);
                emax = max(emax, out & 0xFFu);
            }
            p.maps[t * p.P + ph] = out;
        }
        irr = __reduce_or_sync(kD3Full, (uint32_t)irr) |
              ((uint64_t)__reduce_or_sync(kD3Full, (uint32_t)(irr >> 32)) << 32);
        // do all valid entry phases exit at the same phase?  (fast composition)
        const uint32_t m0 = (vl && xraw != kExitInvalid) ? xraw : kExitInvalid;
        if (m0 != kExitInvalid) {
            emin = min(emin, m0);
            emax = max(emax, m0);
        }
        const uint32_t cmn = __reduce_min_sync(kD3Full, emin);
        const bool nonuni = __reduce_max_sync(kD3Full, emax) != cmn && cmn != kExitInvalid;
        if (lane == 0) {
            p.maps[t * p.P] = m0 == kExitInvalid ? kExitInvalid : ((tot << 8) | xraw);
            p.irr[t] = irr;
            p.uexit[t] = (uint8_t)cmn;
            if (nonuni) atomicAdd(p.nonuni, 1u);
        }
        __syncwarp();
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
}


// count-only decode with the byte LUT (irregular entries in final9)
__device__ __forceinline__ bool d3_count8(const uint32_t *stg, uint32_t head, const uint64_t *s_lut,
                                          const uint16_t *s_st, const uint8_t *s_l1, const DecCanon *tab,
                                          uint32_t mstop, uint32_t &rel, uint32_t &cnt) {
    cnt = 0;
    if (rel >= mstop) return true;
    SWin r;
    r.init(stg, rel + head);
    while (rel < mstop) {
        const uint32_t pk = r.peek12();
        const uint64_t en = s_lut[pk];
        uint32_t n = (uint32_t)(en >> 48) & 7u, adv = (uint32_t)(en >> 51) & 15u;
        if (n == 0) {
            const uint32_t l1 = s_l1[pk];
            adv = (l1 & 0x80u) ? dlen_long(tab, r.peek64(), l1 & 0x7Fu) : l1;
            if (adv == 0) return false;
            n = 1;
        } else if (mstop - rel < (uint32_t)kLutBits) {
            const uint32_t hs = (uint32_t)s_st[pk] & (0xFFFu << (mstop - rel));
            n -= __popc(hs);
            adv = hs ? (uint32_t)(__ffs(hs) - 1) : adv;
        }
        cnt += n;
        rel += adv;
        r.skip(adv);
    }
    return true;
}

// Final decode with a byte-wide stage (u16 books): symbols are staged as
// bytes s - (cap/2 - 128) and widened in the copy-out, and the decode LUT
// holds byte deltas (8-byte entries), so a warp needs half the shared memory
// of a u16 stage (the earlier k_dec_final7) and twice as many warps fit on an SM (the single-chain
// decode is latency-bound).  A symbol outside the byte range (rare: such
// symbols have long code words) is staged as the escape byte 255 and its
// value kept in a per-warp side list that patches the output after the
// copy-out; a subsequence with more than kF9Esc of them is re-decoded with
// u16 stores straight to global memory.
constexpr int kF9Warps = 32;
constexpr uint32_t kF9Stage = 4256;  // bytes per warp: <= 4096 + 7 (alignment) + overrun slack
constexpr uint32_t kF9Esc = 16;      // escaped symbols per warp and subsequence

__global__ void __launch_bounds__(kF9Warps * 32, 1) k_dec_final9(DecParams p, uint32_t cap) {
    extern __shared__ __align__(16) unsigned char f9_smem[];
    uint64_t *s_lut = reinterpret_cast<uint64_t *>(f9_smem);
    uint16_t *s_st = reinterpret_cast<uint16_t *>(s_lut + kLutSize);
    uint16_t *s_s1 = s_st + kLutSize;
    uint8_t *s_l1 = reinterpret_cast<uint8_t *>(s_s1 + kLutSize);
    uint8_t *s_out = s_l1 + kLutSize;                                               // kF9Warps * kF9Stage
    uint32_t *s_str = reinterpret_cast<uint32_t *>(s_out + kF9Warps * kF9Stage);   // kF9Warps * 2 * kStgWords
    __shared__ DecCanon s_can;
    __shared__ uint32_t s_esc[kF9Warps][kF9Esc];  // stage index << 16 | symbol
    __shared__ uint32_t s_nesc[kF9Warps];
    for (uint32_t i = threadIdx.x; i < kLutSize; i += blockDim.x) {
        s_lut[i] = p.tab->lut8[i];
        s_st[i] = p.tab->lut8s[i];
        s_s1[i] = p.tab->lut1s[i];
        s_l1[i] = p.tab->lut1[i];
    }
    load_canon(s_can, p.tab);
    __syncthreads();
    if (p.st->code) return;  // corrupt stream: leave the output untouched
    const DecCanon *tab = &s_can;
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    // table addresses held in registers (otherwise the shared window base is
    // rebuilt from SR_CgaCtaId inside the decode loop: 4 instructions a step)
    const uint32_t lut_s = smem_addr(s_lut), st_s = smem_addr(s_st), s1_s = smem_addr(s_s1),
                   l1_s = smem_addr(s_l1);
    const int32_t base8 = (int32_t)(cap / 2) - 128;
    const uint32_t b2 = ((uint32_t)base8 & 0xFFFFu) * 0x00010001u;  // per-halfword widening addend
    uint8_t *wout = s_out + warp * kF9Stage;
    const uint32_t out_s = (uint32_t)__cvta_generic_to_shared(wout);
    uint32_t *wstr = s_str + warp * 2 * kStgWords;
    const uint32_t str_s = (uint32_t)__cvta_generic_to_shared(wstr);
    uint16_t *out = static_cast<uint16_t *>(p.out);
    const uint64_t nw = (uint64_t)gridDim.x * kF9Warps;
    uint64_t t = (uint64_t)blockIdx.x * kF9Warps + warp;
    uint32_t sb = 0;
    d3_stage(p, t, str_s, lane);
    for (; t < p.T; t += nw, sb ^= 1) {
        d3_stage(p, t + nw, str_s + (sb ^ 1) * kStgWords * 4, lane);
        d3_stage_wait();
        const uint32_t *stg = wstr + sb * kStgWords;
        const bool plan = p.psoff != nullptr;
        const uint32_t e = plan ? (p.cp[t * 32] & 0xFFu) : p.ent0[t];
        if (e == kExitInvalid || e == kExitEnd) continue;
        const uint64_t t0 = t * kS3;
        const bool last = t == p.T - 1;
        const uint32_t stop = last ? (uint32_t)(p.bit_len - t0) : kS3;
        const uint32_t la = (stop + kMB - 1) / kMB - 1;
        const uint64_t base = plan ? p.psoff[t] : p.off0[t];
        const uint64_t endo = last ? p.count : plan ? p.psoff[t + 1] : p.off0[t + 1];
        const uint32_t total = (uint32_t)(endo - base);
        const uint32_t b = lane * kMB;
        const bool act = lane <= la;
        const uint32_t mstop = act ? min(b + kMB, stop) : b;
        const uint32_t cpv = act ? p.cp[t * 32 + lane] : 0u;
        uint32_t cnt = act ? (cpv >> 8) : 0u;
        uint32_t start = act ? b + (cpv & 0xFFu) : b;
        if (lane == 0) start = e;
        const bool irregular = plan ? p.pirr[t] != 0 : (e != 0 && ((p.irr[t] >> e) & 1ull));
        if (irregular) {
            // the true path joins the chain after microblock 0: re-resolve the
            // lanes' starts and counts (count-only, lane by lane)
            uint32_t x = __shfl_down_sync(kD3Full, start, 1);  // chain exit guess
            bool need = lane == 0;
            bool bad = false;
            while (__any_sync(kD3Full, need)) {
                bool changed = false;
                if (need && act) {
                    uint32_t rel = start, c;
                    if (!d3_count8(stg, p.head, s_lut, s_st, s_l1, tab, mstop, rel, c)) bad = true;
                    changed = rel != x;
                    cnt = c;
                    x = rel;
                }
                const uint32_t px = __shfl_up_sync(kD3Full, x, 1);
                const bool pc = __shfl_up_sync(kD3Full, changed, 1);
                need = lane > 0 && act && pc && px != start;
                if (need) start = px;
            }
            if (__any_sync(kD3Full, bad)) {
                if (lane == 0) set_status(p.st, LZB_E_CORRUPT);
                continue;
            }
        } else {
            const uint32_t rest = __reduce_add_sync(kD3Full, lane ? cnt : 0u);
            if (lane == 0) cnt = total - rest;
        }
        uint32_t inc = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(kD3Full, inc, o);
            if (lane >= (uint32_t)o) inc += v;
        }
        const uint32_t pre = inc - cnt;
        const uint32_t sum = __shfl_sync(kD3Full, inc, 31);
        // stage byte j <-> output element base - sh + j; out + base - sh is 16-byte aligned
        const uint32_t sh = (uint32_t)(((reinterpret_cast<uintptr_t>(out) >> 1) + base) & 7u);
        bool bad = sum != total || total > kS3 || (act && cnt > kMB);
        bool wide = false;  // more escaped symbols than the side list holds
        if (lane == 0) s_nesc[warp] = 0;
        __syncwarp();
        uint32_t rel = start;
        const uint32_t a0 = out_s + sh + pre;  // the lane's first stage byte
        uint32_t a = a0;
        if (!__any_sync(kD3Full, bad) && act && rel < mstop) {
            SWin r;
            r.init(stg, rel + p.head);
            while (rel < mstop) {
                const uint32_t pk = r.peek12();
                uint32_t lo, hi;
                asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(lut_s + 8 * pk));
                uint32_t n = (hi >> 16) & 7u, adv = (hi >> 19) & 15u;
                if (n == 0) {  // long code word, out-of-byte symbol, or invalid prefix
                    const uint32_t l1 = lds8(l1_s + pk);
                    uint32_t sym = 0;
                    if (l1 & 0x80u) adv = dsym_long(tab, p.syms, r.peek64(), l1 & 0x7Fu, sym);
                    else if (l1) {
                        adv = l1;
                        sym = lds16(s1_s + 2 * pk);
                    } else {
                        adv = 0;
                    }
                    if (adv == 0) {
                        bad = true;
                        break;
                    }
                    const int32_t d = (int32_t)sym - base8;
                    if (d < 0 || d > 254) {  // escape: the value goes to the side list
                        const uint32_t k = atomicAdd(&s_nesc[warp], 1u);
                        if (k < kF9Esc) s_esc[warp][k] = ((a - out_s) << 16) | sym;
                        else wide = true;
                        lo = 255u;
                    } else {
                        lo = (uint32_t)d;
                    }
                    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(lo) : "memory");
                    a += 1;
                    rel += adv;
                    r.skip(adv);  // a long code word may exceed 32 bits
                    continue;
                }
                if (mstop - rel < (uint32_t)kLutBits) {  // code words must start before mstop
                    const uint32_t hs = lds16(st_s + 2 * pk) & (0xFFFu << (mstop - rel));
                    n -= __popc(hs);
                    adv = hs ? (uint32_t)(__ffs(hs) - 1) : adv;
                }
                // predicated (not branched) byte stores: one per decoded symbol
                asm volatile(
                    "{\n\t.reg .pred q1, q2, q3, q4, q5;\n\t"
                    "setp.gt.u32 q1, %3, 1;\n\tsetp.gt.u32 q2, %3, 2;\n\tsetp.gt.u32 q3, %3, 3;\n\t"
                    "setp.gt.u32 q4, %3, 4;\n\tsetp.gt.u32 q5, %3, 5;\n\t"
                    "st.shared.u8 [%0], %1;\n\t"
                    "@q1 st.shared.u8 [%0+1], %4;\n\t"
                    "@q2 st.shared.u8 [%0+2], %5;\n\t"
                    "@q3 st.shared.u8 [%0+3], %6;\n\t"
                    "@q4 st.shared.u8 [%0+4], %2;\n\t"
                    "@q5 st.shared.u8 [%0+5], %7;\n\t}"
                    ::"r"(a), "r"(lo), "r"(hi), "r"(n), "r"(lo >> 8), "r"(lo >> 16), "r"(lo >> 24), "r"(hi >> 8)
                    : "memory");
                a += n;
                rel += adv;
                r.consume(adv);  // <= 12 bits from the LUT
            }
        }
        if (__any_sync(kD3Full, wide) && !__any_sync(kD3Full, bad)) {
            // u16 symbols straight to global memory (slow path)
            rel = start;
            uint64_t o = base + pre;
            const uint64_t o0 = o;
            if (act && rel < mstop) {
                SWin r;
                r.init(stg, rel + p.head);
                while (rel < mstop) {
                    const uint32_t pk = r.peek12();
                    const uint32_t l1 = s_l1[pk];
                    uint32_t sym = 0, L;
                    if (l1 & 0x80u) L = dsym_long(tab, p.syms, r.peek64(), l1 & 0x7Fu, sym);
                    else {
                        L = l1;
                        sym = s_s1[pk];
                    }
                    if (L == 0 || o - o0 >= cnt) {
                        bad = true;
                        break;
                    }
                    out[o++] = (uint16_t)sym;
                    rel += L;
                    r.skip(L);
                }
            }
            if (act && o - o0 != cnt) bad = true;
            const uint32_t nstart = __shfl_down_sync(kD3Full, start, 1);
            if (act && lane < la && rel != nstart) bad = true;
            if (__any_sync(kD3Full, bad) && lane == 0) set_status(p.st, LZB_E_CORRUPT);
            continue;
        }
        if (act && (a - a0) != cnt) bad = true;
        {
            const uint32_t nstart = __shfl_down_sync(kD3Full, start, 1);
            if (act && lane < la && rel != nstart) bad = true;
        }
        if (__any_sync(kD3Full, bad)) {
            if (lane == 0) set_status(p.st, LZB_E_CORRUPT);
            continue;
        }
        __syncwarp();
        // copy-out: 8 staged bytes -> 8 u16 symbols (one 16-byte store)
        const uint64_t g0 = base - sh;
        const uint32_t q0 = sh ? 1u : 0u, q1 = (sh + total) >> 3;
        const uint2 *wv = reinterpret_cast<const uint2 *>(wout);
        for (uint32_t q = q0 + lane; q < q1; q += 32) {
            const uint2 v = wv[q];
            uint4 w;
            w.x = __vadd2(__byte_perm(v.x, 0u, 0x4140), b2);
            w.y = __vadd2(__byte_perm(v.x, 0u, 0x4342), b2);
            w.z = __vadd2(__byte_perm(v.y, 0u, 0x4140), b2);
            w.w = __vadd2(__byte_perm(v.y, 0u, 0x4342), b2);
            *reinterpret_cast<uint4 *>(out + g0 + 8 * q) = w;
        }
        {  // the partial head / tail units, one element per lane
            const uint32_t c = lane & 7;
            const uint32_t j = (lane < 8 ? 0u : 8u * q1) + c;
            const bool part = lane < 8 ? (sh != 0) : (lane < 16 && ((sh + total) & 7) != 0);
            if (part && j >= sh && j < sh + total) out[g0 + j] = (uint16_t)((int32_t)wout[j] + base8);
        }
        __syncwarp();
        {  // patch the escaped symbols over their widened escape bytes
            const uint32_t ne = s_nesc[warp];
            for (uint32_t k = lane; k < ne; k += 32) {
                const uint32_t v = s_esc[warp][k];
                out[g0 + (v >> 16)] = (uint16_t)(v & 0xFFFFu);
            }
        }
        __syncwarp();
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
}
