/*
 * lzb.h -- C ABI of liblzb.so, the B200 (sm_100a) implementation of the
 * cuSZ+ / lzebc compress-decompress hot path.
 *
 * The reference (lzebc, a Python package) has no native boundary: its hot path
 * is a set of Python functions.  Each entry point below replaces one of them;
 * the replaced reference interface is cited as P/<file>:<line> with
 * P = /root/reference/pkg/src/lzebc/.  A host binding (ctypes, the one this
 * repo ships in paper_2105_12912_b200/_native.py) calls these with plain
 * device pointers; see INTEGRATION.md for the binding a reference maintainer
 * would add.
 *
 * Conventions
 *  - Every pointer named x/y/sym/codes/hist/out/... is a DEVICE pointer
 *    (cudaMalloc'd or a torch CUDA tensor's data_ptr()).  `stream` is a
 *    cudaStream_t passed as void*; NULL = legacy default stream.
 *  - All calls are asynchronous on `stream`.  The return value reports only
 *    argument and launch errors.  Data-dependent outcomes (overflow, corrupt
 *    archive, non-finite values, sizes) are written to the DEVICE status block
 *    `st`, which the host reads at its single synchronisation point.
 *  - The caller owns all memory, including scratch (size from the matching
 *    *_scratch_bytes query).  The library holds no global mutable state, so
 *    calls on distinct streams with distinct buffers may run concurrently.
 *  - Results are deterministic: integer atomics only into order-independent
 *    sums; no floating-point atomics.
 *  - dtype: 0 = float32, 1 = float64.  Symbol/code width: 2 (u16, cap <= 65536)
 *    or 4 (u32) bytes.
 */
#ifndef LZB_H
#define LZB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; map onto P/errors.py:4-17 */
#define LZB_OK 0
#define LZB_E_ARG 1        /* bad argument / scratch too small (caller bug)    */
#define LZB_E_DATA 2       /* DataError                                        */
#define LZB_E_OVERFLOW 3   /* QuantOverflowError                               */
#define LZB_E_CORRUPT 4    /* CorruptArchiveError                              */
#define LZB_E_CUDA 5       /* CUDA launch / runtime error                      */
#define LZB_E_ASSERT 6     /* the reference's debug assert (P/quantize.py:106) */
#define LZB_E_CAPACITY 7   /* output buffer too small; true size in st->u[..]  */
#define LZB_E_RETRY 8      /* fast decoder could not resolve the stream: call  */
                           /* lzb_huff_decode_robust (also judges corruption)  */

/* Dims + ChunkSpec (P/grid.py:27-93) */
typedef struct lzb_geom {
    uint64_t nx, ny, nz; /* extents, x fastest                        */
    uint64_t cx, cy, cz; /* chunk edges                               */
    int32_t ndim;        /* 1, 2 or 3 (Lorenzo order, P/grid.py:31-33) */
    int32_t reserved;
} lzb_geom;

/* Device status block.  code: first error (LZB_*), 0 if none. */
typedef struct lzb_dstatus {
    int32_t code;
    int32_t detail;
    uint64_t u[6]; /* op-specific results, documented per entry point */
} lzb_dstatus;

const char *lzb_version(void);
const char *lzb_strerror(int code);

/* Byte copy executed by SMs rather than a copy engine (host utility, not a
 * reference stage): with unified addressing either pointer may be pinned
 * host memory, so a small host<->device copy issued this way runs beside
 * large DMA transfers instead of queueing behind them. */
int lzb_copy_bytes(void *dst, const void *src, uint64_t n, void *stream);

/* ---------------------------------------------------------------------
 * Field range + finiteness.  Replaces Field.from_array / ingest's
 * min/max/_check_finite (P/grid.py:155-202).
 * st->u[0] = vmin (f64 bits), u[1] = vmax (f64 bits),
 * u[2] = first non-finite element offset or UINT64_MAX; code = LZB_E_DATA
 * if any element is non-finite.
 * ------------------------------------------------------------------- */
int lzb_field_range(const void *x, int dtype, uint64_t n, lzb_dstatus *st, void *stream);

/* ---------------------------------------------------------------------
 * Prequantization only (P/quantize.py:95-110):
 * out[i] = trunc(q + copysign(0.5, q)), q = f64(x[i]) / (2*eb_abs).
 * code = LZB_E_OVERFLOW if any |out| >= 2^59, LZB_E_ASSERT if the bound
 * invariant fails.
 * ------------------------------------------------------------------- */
int lzb_prequantize(const void *x, int dtype, uint64_t n, double eb_abs, int64_t *out,
                    lzb_dstatus *st, void *stream);

/* ---------------------------------------------------------------------
 * Verification hook for K1's fast prequantizers (the f32 double-single and
 * f64 magic-number paths that replace the reference's f64 division,
 * P/quantize.py:95-110).  dtype 0: the f32 bit patterns [lo, lo + count);
 * dtype 1: `count` f64 values from hashed bit patterns starting at lo.
 * st->u[0] = fast results that disagree with the exact rule (must be 0),
 * u[1] = inputs the fast path accepted, u[2] = finite inputs examined.
 * ------------------------------------------------------------------- */
int lzb_prequant_verify(double eb_abs, uint64_t lo, uint64_t count, int dtype, lzb_dstatus *st,
                        void *stream);

/* ---------------------------------------------------------------------
 * K1: fused prequantize + Lorenzo delta + quant code + histogram +
 * outlier gather, emitting the CHUNK-MAJOR symbol stream.
 * Replaces prequantize + construct_grid + gather_chunk_major + histogram
 * (P/quantize.py:90-213, P/pipeline.py:102-105, P/codebook.py:23-27).
 *   codes     : n symbols, chunk-major, width code_bytes (naturally aligned;
 *               a 16-byte aligned buffer enables the register fast paths
 *               for ChunkSpec 8x8x8 / 16x16 / 256, else the generic path)
 *   hist      : cap x u64, OVERWRITTEN with the stream histogram
 *   outliers  : out_capacity records of {u64 index, i64 delta}, sorted by
 *               global row-major index (the archive's outlier section)
 * dtype may also be 2 = int64 prequant integers (construct_grid on a
 * PrequantGrid, P/quantize.py:161): prequantization is then skipped.
 * st->u[0] = outlier count.  If it exceeds out_capacity the records are not
 * complete and code = LZB_E_CAPACITY (retry with a larger buffer).
 * ------------------------------------------------------------------- */
size_t lzb_quantize_scratch_bytes(const lzb_geom *g, uint64_t out_capacity);
int lzb_quantize(const void *x, int dtype, const lzb_geom *g, double eb_abs, uint32_t cap,
                 void *codes, int code_bytes, uint64_t *hist, uint64_t *outliers,
                 uint64_t out_capacity, lzb_dstatus *st, void *scratch, size_t scratch_bytes,
                 void *stream);

/* lzb_quantize that also records `hist_event` (a cudaEvent_t; may be NULL)
 * on the stream as soon as `hist` is final -- before the outlier compaction
 * and ordering launches -- so the code book (K2) can be built on a second
 * stream while they run. */
int lzb_quantize_ev(const void *x, int dtype, const lzb_geom *g, double eb_abs, uint32_t cap,
                    void *codes, int code_bytes, uint64_t *hist, uint64_t *outliers,
                    uint64_t out_capacity, lzb_dstatus *st, void *scratch, size_t scratch_bytes,
                    void *stream, void *hist_event);

/* ---------------------------------------------------------------------
 * Histogram of a symbol stream (P/codebook.py:23-27).  hist (cap x u64) is
 * overwritten.  code = LZB_E_DATA if a symbol >= cap (u[0] = that symbol).
 * ------------------------------------------------------------------- */
int lzb_histogram(const void *sym, int sym_bytes, uint64_t n, uint32_t cap, uint64_t *hist,
                  lzb_dstatus *st, void *stream);

/* ---------------------------------------------------------------------
 * K2: canonical Huffman code book from a histogram.  Replaces
 * Codebook.from_counts (_huffman_lengths + _canonical_codes,
 * P/codebook.py:120-123, 143-190) and the exact <b> of select_workflow
 * (P/codebook.py:110-115, P/smoothness.py:111-136).
 *   lengths : cap x u8, codes : cap x u64 (MSB-first code words)
 * st->u[0] = sum(count*len), u[1] = total count, u[2] = max length,
 * u[3] = symbols used.  code = LZB_E_DATA on an empty histogram or a code
 * longer than 64 bits.
 * ------------------------------------------------------------------- */
size_t lzb_codebook_scratch_bytes(uint32_t cap);
int lzb_codebook(const uint64_t *hist, uint32_t cap, uint8_t *lengths, uint64_t *codes,
                 lzb_dstatus *st, void *scratch, size_t scratch_bytes, void *stream);

/* ---------------------------------------------------------------------
 * Canonical code words from serialized lengths + validation.  Replaces
 * Codebook.from_lengths (P/codebook.py:125-140).  code = LZB_E_CORRUPT on a
 * length > 64, an empty book, a bad single-symbol book, or Kraft inequality.
 * st->u[2] = max length, u[3] = symbols used.
 * ------------------------------------------------------------------- */
int lzb_codebook_from_lengths(const uint8_t *lengths, uint32_t cap, uint64_t *codes,
                              lzb_dstatus *st, void *scratch, size_t scratch_bytes, void *stream);

/* ---------------------------------------------------------------------
 * K3: Huffman bit packing (P/huffman.py:46-61).  Writes exactly
 * ceil(bit_len/8) bytes at `out` (MSB first, last byte zero padded); out
 * need not be aligned.  out_bytes must be >= ceil(bit_len/8) where bit_len =
 * sum(len(sym)) (known beforehand from lzb_codebook's u[0]).  maxlen = the
 * book's longest code word (lzb_codebook's u[2]; 0 = unknown, generic path;
 * LZB_MAXLEN_DEVICE = the book is built by lzb_codebook earlier in the same
 * stream and not read back: 16-bit symbols, cap <= 4096, buffers sized for
 * 32-bit code words, code = LZB_E_RETRY if the book has a longer one -- the
 * output is then unusable and the caller re-runs with the true maxlen).
 * st->u[0] = bit_len.  code = LZB_E_DATA if a symbol has no code word.
 * ------------------------------------------------------------------- */
#define LZB_MAXLEN_DEVICE 0xFFFFFFFFu
size_t lzb_huff_encode_scratch_bytes(uint64_t n);
int lzb_huff_encode(const void *sym, int sym_bytes, uint64_t n, const uint8_t *lengths,
                    const uint64_t *codes, uint32_t cap, uint32_t maxlen, uint8_t *out,
                    uint64_t out_bytes, lzb_dstatus *st, void *scratch, size_t scratch_bytes,
                    void *stream);

/* Device-side assembly of a Huffman archive (single-sync compress; archive
 * layout of P/pipeline.py:184-221).  `header` (host, 130 bytes) is the packed
 * header with everything but outlier_count, sym_len, out_off and out_len,
 * which come from st_quant->u[0] (K1's outlier count) and st_book->u[0]
 * (K2's bit length).  Writes the header, the code lengths at 136, the
 * [bit_len][count] prefix at sym_off (= align8(136 + cap); the bit stream
 * itself is written by lzb_huff_encode at sym_off + 16), the zero padding
 * and the 16-byte outlier records.  st->u[0] = total archive bytes,
 * st->u[1] = out_off; code = LZB_E_CAPACITY if total > arc_bytes (nothing
 * written).  Does nothing if st_quant or st_book carries an error. */
int lzb_archive_finalize_huff(uint8_t *arc, uint64_t arc_bytes, const uint8_t *header, uint64_t sym_off,
                              const uint8_t *lengths, uint32_t cap, const lzb_dstatus *st_quant,
                              const lzb_dstatus *st_book, const void *records, lzb_dstatus *st,
                              void *stream);

/* Multi-GPU slab variant of lzb_huff_encode: the first bit lands at bit
 * `bit_offset` (0..7, MSB first) of out[0]; bits outside the slab are zero so
 * neighbouring slabs OR-merge their shared boundary byte. */
int lzb_huff_encode_at(const void *sym, int sym_bytes, uint64_t n, const uint8_t *lengths,
                       const uint64_t *codes, uint32_t cap, uint32_t maxlen, uint64_t bit_offset,
                       uint8_t *out, uint64_t out_bytes, lzb_dstatus *st, void *scratch,
                       size_t scratch_bytes, void *stream);

/* ---------------------------------------------------------------------
 * K5: self-synchronising parallel Huffman decode of a dense MSB-first bit
 * stream (replaces lzebc.huffman.decode, P/huffman.py:64-122, and its numba
 * kernel _decode_kernel, P/huffman.py:85-106).  `bits` holds ceil(bit_len/8)
 * bytes, any alignment.  Writes `count` symbols.  `maxlen` is the largest
 * entry of `lengths` (the host reads it from the archive's code book
 * section; the device re-checks it).  code = LZB_E_CORRUPT for an invalid
 * code book (Codebook.from_lengths rules) or when the stream does not decode
 * to exactly `count` code words ending at bit_len.
 *
 * lzb_huff_decode is the fast two-pass decoder (u16 symbols): it may end with
 * code = LZB_E_RETRY instead (a book that does not resynchronise within a
 * 128-bit microblock, or any irregular/corrupt stream); the caller then runs
 * lzb_huff_decode_robust on the same arguments, the exhaustive decoder
 * (transfer maps of every entry phase), which also reports corruption.
 * ------------------------------------------------------------------- */
size_t lzb_huff_decode_scratch_bytes(uint64_t bit_len, uint32_t maxlen, uint32_t cap);
int lzb_huff_decode(const uint8_t *bits, uint64_t bit_len, uint64_t count,
                    const uint8_t *lengths, uint32_t cap, uint32_t maxlen, void *sym,
                    int sym_bytes, lzb_dstatus *st, void *scratch, size_t scratch_bytes,
                    void *stream);
int lzb_huff_decode_robust(const uint8_t *bits, uint64_t bit_len, uint64_t count,
                           const uint8_t *lengths, uint32_t cap, uint32_t maxlen, void *sym,
                           int sym_bytes, lzb_dstatus *st, void *scratch, size_t scratch_bytes,
                           void *stream);

/* Multi-GPU slab variant: the stream's first bit is bit
 * `bit_phase` (0..7, MSB first) of bits[0] -- a rank's slice as produced by
 * lzb_huff_encode_at.  Same outputs and errors as lzb_huff_decode. */
int lzb_huff_decode_at(const uint8_t *bits, uint64_t bit_phase, uint64_t bit_len, uint64_t count,
                       const uint8_t *lengths, uint32_t cap, uint32_t maxlen, void *sym,
                       int sym_bytes, lzb_dstatus *st, void *scratch, size_t scratch_bytes,
                       void *stream);

/* ---------------------------------------------------------------------
 * Bit-range decode: multi-GPU decompression of ONE stored stream (SURVEY
 * §8e; the reference decodes the whole stream in one process,
 * P/huffman.py:107-138).  A rank owns stream bits [bit_lo, bit_hi) of the
 * stream at `bits` (4-byte aligned, bit_len bits in total, replicated on
 * every rank); bit_lo is a multiple of LZB_DEC_RANGE_ALIGN and bit_hi is
 * too unless it is bit_len.
 *
 * lzb_huff_range_maps writes fmap[p] = (symbols << 8) | exit for every
 * entry phase p < maxlen: decoding the range from bit bit_lo + p yields
 * `symbols` code words and leaves at phase `exit` of the next range (0xFE:
 * the stream ended exactly, 0xFF: invalid).  The host chains the ranks'
 * maps from phase 0 to get each range's entry phase, exit phase and symbol
 * count; lzb_huff_range_decode (same scratch, still holding pass 1's state)
 * then writes the range's `count` symbols.  A chain that does not end in
 * 0xFE with the header's symbol count is a corrupt archive.
 * ------------------------------------------------------------------- */
#define LZB_DEC_RANGE_ALIGN 4096
size_t lzb_huff_range_scratch_bytes(uint64_t range_bits, uint32_t maxlen, uint32_t cap);
int lzb_huff_range_maps(const uint8_t *bits, uint64_t bit_len, uint64_t bit_lo, uint64_t bit_hi,
                        const uint8_t *lengths, uint32_t cap, uint32_t maxlen, uint64_t *fmap,
                        lzb_dstatus *st, void *scratch, size_t scratch_bytes, void *stream);
int lzb_huff_range_decode(const uint8_t *bits, uint64_t bit_len, uint64_t bit_lo, uint64_t bit_hi,
                          const uint8_t *lengths, uint32_t cap, uint32_t maxlen, uint32_t entry,
                          uint32_t exit_phase, uint64_t count, void *sym, int sym_bytes,
                          lzb_dstatus *st, void *scratch, size_t scratch_bytes, void *stream);

/* ---------------------------------------------------------------------
 * Number of maximal runs of a symbol stream (sizes K4's outputs before the
 * RLE / RLE_VLE workflows, P/rle.py:17-35).  st->u[0] = run count.
 * ------------------------------------------------------------------- */
int lzb_count_runs(const void *sym, int sym_bytes, uint64_t n, lzb_dstatus *st, void *stream);

/* ---------------------------------------------------------------------
 * K4: run-length encode (P/rle.py:17-35): maximal runs, runs longer than
 * max_run (0xFFFFFFFF in the reference) split.  values/lengths: u32.
 * st->u[0] = run count; code = LZB_E_CAPACITY if > cap_runs.
 * ------------------------------------------------------------------- */
size_t lzb_rle_encode_scratch_bytes(uint64_t n);
int lzb_rle_encode(const void *sym, int sym_bytes, uint64_t n, uint32_t *values,
                   uint32_t *lengths, uint64_t cap_runs, uint64_t max_run, lzb_dstatus *st,
                   void *scratch, size_t scratch_bytes, void *stream);

/* ---------------------------------------------------------------------
 * K7: run-length decode (P/rle.py:38-44, P/pipeline.py:283-302).  values
 * and lengths are little-endian u32 arrays at ANY byte alignment (the
 * RLE_VLE lengths array is unaligned in the archive).  Validates zero-length
 * runs, sum(lengths) == n and value < cap BEFORE expanding
 * (code = LZB_E_CORRUPT).
 * ------------------------------------------------------------------- */
size_t lzb_rle_decode_scratch_bytes(uint64_t runs);
int lzb_rle_decode(const uint8_t *values_le, const uint8_t *lengths_le, uint64_t runs,
                   uint32_t cap, void *sym, int sym_bytes, uint64_t n, lzb_dstatus *st,
                   void *scratch, size_t scratch_bytes, void *stream);

/* ---------------------------------------------------------------------
 * K6: fused outlier fuse + chunk-wise multi-dimensional partial-sum
 * reconstruction + dequantization + range/finiteness.  Replaces
 * scatter_chunk_major + _decode_outliers validation + reconstruct_grid +
 * dequantize (P/pipeline.py:108-117, 306-315, P/reconstruct.py:22-88).
 *   codes    : chunk-major symbols (naturally aligned; full chunks of a
 *              16-byte aligned stream are read with vector loads)
 *   outliers : n_out 16-byte LE records {u64 index, i64 delta}, any alignment
 *   y        : n values (dtype) in grid (row-major) order
 * st->u[0]/u[1] = vmin/vmax (f64 bits), u[2] = first non-finite offset.
 * code = LZB_E_CORRUPT for a bad outlier list, LZB_E_OVERFLOW for the
 * prefix-sum guard, LZB_E_DATA for a non-finite value.
 * ------------------------------------------------------------------- */
size_t lzb_reconstruct_scratch_bytes(const lzb_geom *g, uint64_t n_out);
int lzb_reconstruct(const void *codes, int code_bytes, const uint8_t *outliers, uint64_t n_out,
                    const lzb_geom *g, double eb_abs, uint32_t cap, void *y, int dtype,
                    int64_t *prequant_out, lzb_dstatus *st, void *scratch,
                    size_t scratch_bytes, void *stream);

/* Dequantization only (P/reconstruct.py:79-88): y = dtype(f64(q) * 2 eb_abs);
 * st as for lzb_reconstruct (range, first non-finite offset, LZB_E_DATA). */
int lzb_dequantize(const int64_t *q, uint64_t n, double eb_abs, void *y, int dtype,
                   lzb_dstatus *st, void *stream);

/* ---------------------------------------------------------------------
 * Grid <-> chunk-major reorder of 2- or 4-byte elements
 * (gather_chunk_major / scatter_chunk_major, P/pipeline.py:102-117).
 * direction 0 = gather (grid -> stream), 1 = scatter (stream -> grid).
 * ------------------------------------------------------------------- */
int lzb_chunk_major(const void *src, void *dst, int elem_bytes, const lzb_geom *g,
                    int direction, void *stream);

/* ---------------------------------------------------------------------
 * Quality statistics (P/pipeline.py:329-345): st->u[0] = max |a-b| (f64
 * bits), u[1] = sum (a-b)^2 (f64 bits, deterministic order).
 * ------------------------------------------------------------------- */
size_t lzb_quality_scratch_bytes(uint64_t n);
int lzb_quality(const void *a, const void *b, int dtype, uint64_t n, lzb_dstatus *st,
                void *scratch, size_t scratch_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* LZB_H */
