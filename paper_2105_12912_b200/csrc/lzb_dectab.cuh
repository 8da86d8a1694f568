// Decode tables shared by the K5 decoders (lzb_huff.cu) and the fused
// decode + reconstruct kernel (lzb_recon.cu): canonical tables of the code
// book (P/huffman.py:64-82) and the 12-bit multi-code-word LUTs built from
// them by k_dec_tables / k_dec_luts.
#pragma once

#include "lzb_common.cuh"

namespace lzb {

constexpr int kLutBits = 12;
constexpr uint32_t kLutSize = 1u << kLutBits;
constexpr uint8_t kExitInvalid = 0xFF;
constexpr uint8_t kExitEnd = 0xFE;

struct DecTables {
    // Multi-symbol LUT on the next 12 bits: up to three complete code words
    // greedily decoded from the window.  bits 0-1 count (0 = first code word
    // longer than 12 bits or invalid prefix), 2-5/6-9/10-13 their lengths,
    // 16-31/32-47/48-63 their symbols (books with cap > 65536 use count 0).
    uint64_t lutm[kLutSize];
    uint8_t lut1[kLutSize];  // first code word: len <= 12, or 0x80 | shortest long len, 0 invalid
    // Byte LUT for the final decode (u16 books, symbols near the radius):
    // up to six code words whose symbols s satisfy 0 <= s - (cap/2 - 128) < 255,
    // stored as those byte deltas; bits 48-50 count (0: first code word longer
    // than 12 bits, invalid, or its symbol out of byte range), 51-54 bits used.
    uint64_t lut8[kLutSize];
    uint16_t lut8s[kLutSize];  // code-word start mask of lut8's code words
    uint16_t lut1s[kLutSize];  // symbol of the first code word (when <= 12 bits)
    // Boundary LUT for the map pass: n | used << 4 | starts << 8, where bit i
    // of `starts` marks a code word starting at window offset i (up to 12
    // complete code words greedily decoded from the 12-bit window).
    uint32_t lutb[kLutSize];
    // Count LUT for K5 v4's map pass: used bits | count << 16 of all complete
    // code words in the window; 0x80000000 when the first is longer than the
    // LUT or invalid (one add advances position and count together).
    uint32_t lutc[kLutSize];
    // Symbol LUT for K5 v4's tile decoder (u16 books): up to six complete code
    // words as u16 symbols in x..z (two per word), w = count | used bits << 8;
    // count 0 = first code word longer than the LUT, or invalid.
    uint4 lut6[kLutSize];
    uint64_t first[65];
    uint64_t cnt[65];
    uint32_t off[65];
    uint32_t maxlen;
    uint32_t nsym;
};

// The canonical tables for code words longer than the LUT, copied to shared
// memory by each decode CTA.
struct DecCanon {
    uint64_t first[65];
    uint64_t cnt[65];
    uint32_t off[65];
    uint32_t maxlen;
};

__device__ __forceinline__ void load_canon(DecCanon &c, const DecTables *t) {
    for (uint32_t i = threadIdx.x; i < 65; i += blockDim.x) {
        c.first[i] = t->first[i];
        c.cnt[i] = t->cnt[i];
        c.off[i] = t->off[i];
    }
    if (threadIdx.x == 0) c.maxlen = t->maxlen;
}

}  // namespace lzb
