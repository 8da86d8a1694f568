/*
 * lzb_oracle.c -- CPU restatement of the reference (lzebc) compress/decompress
 * hot path.  TEST INFRASTRUCTURE ONLY: this file is the parity checker and the
 * timed CPU baseline.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product package never
 * links or calls it.
 *
 * Every function names the reference file:line it restates (paths relative to
 * the reference package root pkg/src/lzebc/).  The arithmetic is restated in
 * plain C on int64 / IEEE binary64 so results are bit-identical with numpy:
 *   - no -ffast-math, no FMA contraction (built with -ffp-contract=off)
 *   - x86-64 SSE2 doubles (IEEE RN)
 *
 * Parity pin: tests/test_oracle_golden.py checks every function here against
 * the golden vectors generated from the reference itself (oracle/gen_golden.py
 * -> tests/golden/).
 *
 * Threading: the chunk loops accept a thread count (OpenMP), mirroring the
 * reference's chunk thread pool (quantize.py:196-205).  Results are
 * independent of the thread count, as in the reference.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_E_OVERFLOW 3   /* QuantOverflowError */
#define ORC_E_ASSERT 6     /* the reference's debug assert (quantize.py:108-111) */
#define ORC_E_CORRUPT 4    /* CorruptArchiveError */
#define ORC_E_DATA 2       /* DataError */
#define ORC_E_NOMEM 7

static const double PREQUANT_LIMIT = 576460752303423488.0; /* 2**59, quantize.py:22 */
static const double PSUM_LIMIT = 4611686018427387904.0;    /* 2**62, reconstruct.py:19 */

static void set_threads(int threads) {
#ifdef _OPENMP
    omp_set_num_threads(threads < 1 ? 1 : threads);
#else
    (void)threads;
#endif
}

/* ---------------------------------------------------------------------------
 * prequantize  (quantize.py:90-110)
 *   scaled = f64(x) / (2*eb_abs); r = trunc(scaled + copysign(0.5, scaled))
 *   any |r| >= 2**59 -> QuantOverflowError; debug assert on the bound.
 * ------------------------------------------------------------------------- */
static int prequant_core(const void *x, int is_f64, int64_t n, double eb_abs,
                         int64_t *out, int threads) {
    const double two_eb = 2.0 * eb_abs;
    const double slack = eb_abs * (1.0 + 1e-12);
    int overflow = 0, assert_fail = 0;
    set_threads(threads);
#pragma omp parallel for schedule(static) reduction(| : overflow, assert_fail)
    for (int64_t i = 0; i < n; i++) {
        double v = is_f64 ? ((const double *)x)[i] : (double)((const float *)x)[i];
        double s = v / two_eb;
        double r = trunc(s + copysign(0.5, s));
        if (fabs(r) >= PREQUANT_LIMIT) {
            overflow = 1;
            out[i] = 0;
            continue;
        }
        int64_t c = (int64_t)r;
        out[i] = c;
        /* assert (abs(values - codes*(2*eb)) <= eb*(1+1e-12)) in f64 */
        if (!(fabs(v - (double)c * two_eb) <= slack)) assert_fail = 1;
    }
    if (overflow) return ORC_E_OVERFLOW;
    if (assert_fail) return ORC_E_ASSERT;
    return ORC_OK;
}

int orc_prequantize(const void *x, int is_f64, int64_t n, double eb_abs, int64_t *out,
                    int threads) {
    return prequant_core(x, is_f64, n, eb_abs, out, threads);
}

/* ---------------------------------------------------------------------------
 * Chunk geometry (grid.py:116-132): chunk ordinals z -> y -> x (x fastest),
 * boundary chunks clipped.  The chunk-major stream (pipeline.py:102-105) is the
 * concatenation of chunks in ordinal order, each row-major inside.
 * ------------------------------------------------------------------------- */
typedef struct {
    int64_t nx, ny, nz, cx, cy, cz;
    int64_t nbx, nby, nbz;
} geom_t;

static geom_t mkgeom(int64_t nx, int64_t ny, int64_t nz, int64_t cx, int64_t cy, int64_t cz) {
    geom_t g = {nx, ny, nz, cx, cy, cz, (nx + cx - 1) / cx, (ny + cy - 1) / cy,
                (nz + cz - 1) / cz};
    return g;
}

/* stream offset of chunk (bx,by,bz): every earlier chunk is fully counted. */
static int64_t chunk_stream_base(const geom_t *g, int64_t bx, int64_t by, int64_t bz) {
    int64_t ez = g->cz < g->nz - bz * g->cz ? g->cz : g->nz - bz * g->cz;
    int64_t ey = g->cy < g->ny - by * g->cy ? g->cy : g->ny - by * g->cy;
    return g->nx * g->ny * g->cz * bz + g->nx * ez * g->cy * by + ez * ey * g->cx * bx;
}

/* gather_chunk_major (pipeline.py:102-105) on u32 grid codes. */
void orc_gather_chunk_major(const uint32_t *grid, int64_t nx, int64_t ny, int64_t nz,
                            int64_t cx, int64_t cy, int64_t cz, uint32_t *stream) {
    geom_t g = mkgeom(nx, ny, nz, cx, cy, cz);
    int64_t pos = 0;
    for (int64_t bz = 0; bz < g.nbz; bz++)
        for (int64_t by = 0; by < g.nby; by++)
            for (int64_t bx = 0; bx < g.nbx; bx++) {
                int64_t x0 = bx * cx, y0 = by * cy, z0 = bz * cz;
                int64_t ex = cx < nx - x0 ? cx : nx - x0;
                int64_t ey = cy < ny - y0 ? cy : ny - y0;
                int64_t ez = cz < nz - z0 ? cz : nz - z0;
                for (int64_t lz = 0; lz < ez; lz++)
                    for (int64_t ly = 0; ly < ey; ly++) {
                        const uint32_t *row = grid + x0 + nx * ((y0 + ly) + ny * (z0 + lz));
                        memcpy(stream + pos, row, (size_t)ex * sizeof(uint32_t));
                        pos += ex;
                    }
            }
}

/* scatter_chunk_major (pipeline.py:108-117). */
void orc_scatter_chunk_major(const uint32_t *stream, int64_t nx, int64_t ny, int64_t nz,
                             int64_t cx, int64_t cy, int64_t cz, uint32_t *grid) {
    geom_t g = mkgeom(nx, ny, nz, cx, cy, cz);
    int64_t pos = 0;
    for (int64_t bz = 0; bz < g.nbz; bz++)
        for (int64_t by = 0; by < g.nby; by++)
            for (int64_t bx = 0; bx < g.nbx; bx++) {
                int64_t x0 = bx * cx, y0 = by * cy, z0 = bz * cz;
                int64_t ex = cx < nx - x0 ? cx : nx - x0;
                int64_t ey = cy < ny - y0 ? cy : ny - y0;
                int64_t ez = cz < nz - z0 ? cz : nz - z0;
                for (int64_t lz = 0; lz < ez; lz++)
                    for (int64_t ly = 0; ly < ey; ly++) {
                        uint32_t *row = grid + x0 + nx * ((y0 + ly) + ny * (z0 + lz));
                        memcpy(row, stream + pos, (size_t)ex * sizeof(uint32_t));
                        pos += ex;
                    }
            }
}

/* ---------------------------------------------------------------------------
 * construct_grid (quantize.py:136-193), emitting the chunk-major stream
 * directly (== gather_chunk_major(construct_grid(...).codes)).
 *
 * Per chunk, delta = nested first differences with zero prepend along the
 * ndim trailing axes (quantize.py:136-141), i.e. the 2^ndim-term Lorenzo
 * stencil restricted to the chunk (zeros outside).  |delta| < r -> code
 * delta + r, else code r and an outlier (global row-major index, delta).
 * Outliers are then sorted by global index (quantize.py:184-193).
 *
 * Returns the outlier count, or -1 if the outlier buffer (cap_out) is too
 * small (call again with a larger buffer).
 * ------------------------------------------------------------------------- */
typedef struct { int64_t idx, delta; } outrec_t;

static int cmp_outrec(const void *a, const void *b) {
    int64_t x = ((const outrec_t *)a)->idx, y = ((const outrec_t *)b)->idx;
    return (x > y) - (x < y);
}

int64_t orc_construct_stream(const int64_t *pre, int64_t nx, int64_t ny, int64_t nz, int ndim,
                             int64_t cx, int64_t cy, int64_t cz, int64_t radius,
                             uint32_t *stream, int64_t *out_idx, int64_t *out_delta,
                             int64_t cap_out, int threads) {
    geom_t g = mkgeom(nx, ny, nz, cx, cy, cz);
    int64_t nchunks = g.nbx * g.nby * g.nbz;
    int64_t total = 0;
    int overflowed = 0;
    outrec_t *recs = (outrec_t *)out_idx; /* scratch view; rewritten below */
    (void)recs;
    /* per-thread outlier vectors */
    int nt = threads < 1 ? 1 : threads;
    outrec_t **tv = (outrec_t **)calloc((size_t)nt, sizeof(outrec_t *));
    int64_t *tn = (int64_t *)calloc((size_t)nt, sizeof(int64_t));
    int64_t *tc = (int64_t *)calloc((size_t)nt, sizeof(int64_t));
    set_threads(nt);
#pragma omp parallel
    {
        int tid = 0;
#ifdef _OPENMP
        tid = omp_get_thread_num();
#endif
#pragma omp for schedule(dynamic, 64)
        for (int64_t c = 0; c < nchunks; c++) {
            int64_t bx = c % g.nbx, by = (c / g.nbx) % g.nby, bz = c / (g.nbx * g.nby);
            int64_t x0 = bx * cx, y0 = by * cy, z0 = bz * cz;
            int64_t ex = cx < nx - x0 ? cx : nx - x0;
            int64_t ey = cy < ny - y0 ? cy : ny - y0;
            int64_t ez = cz < nz - z0 ? cz : nz - z0;
            int64_t pos = chunk_stream_base(&g, bx, by, bz);
            for (int64_t lz = 0; lz < ez; lz++)
                for (int64_t ly = 0; ly < ey; ly++)
                    for (int64_t lx = 0; lx < ex; lx++, pos++) {
                        int64_t gi = (x0 + lx) + nx * ((y0 + ly) + ny * (z0 + lz));
#define V(dz, dy, dx) (((lz) < (dz) || (ly) < (dy) || (lx) < (dx)) ? 0 : \
                        pre[gi - (dx) - nx * ((dy) + ny * (dz))])
                        int64_t d;
                        if (ndim == 1)
                            d = V(0, 0, 0) - V(0, 0, 1);
                        else if (ndim == 2)
                            d = V(0, 0, 0) - V(0, 0, 1) - V(0, 1, 0) + V(0, 1, 1);
                        else
                            d = V(0, 0, 0) - V(0, 0, 1) - V(0, 1, 0) + V(0, 1, 1)
                              - V(1, 0, 0) + V(1, 0, 1) + V(1, 1, 0) - V(1, 1, 1);
#undef V
                        int64_t ad = d < 0 ? -d : d;
                        if (ad < radius) {
                            stream[pos] = (uint32_t)(d + radius);
                        } else {
                            stream[pos] = (uint32_t)radius;
                            if (tn[tid] == tc[tid]) {
                                int64_t nc = tc[tid] ? 2 * tc[tid] : 1024;
                                outrec_t *nv = (outrec_t *)realloc(tv[tid], (size_t)nc * sizeof(outrec_t));
                                if (!nv) { overflowed = 1; continue; }
                                tv[tid] = nv;
                                tc[tid] = nc;
                            }
                            tv[tid][tn[tid]].idx = gi;
                            tv[tid][tn[tid]].delta = d;
                            tn[tid]++;
                        }
                    }
        }
    }
    for (int t = 0; t < nt; t++) total += tn[t];
    int64_t ret = total;
    if (overflowed) ret = -2;
    else if (total > cap_out) ret = -1;
    else {
        outrec_t *all = (outrec_t *)malloc((size_t)(total ? total : 1) * sizeof(outrec_t));
        int64_t k = 0;
        for (int t = 0; t < nt; t++) {
            if (tn[t]) memcpy(all + k, tv[t], (size_t)tn[t] * sizeof(outrec_t));
            k += tn[t];
        }
        qsort(all, (size_t)total, sizeof(outrec_t), cmp_outrec);
        for (int64_t i = 0; i < total; i++) {
            out_idx[i] = all[i].idx;
            out_delta[i] = all[i].delta;
        }
        free(all);
    }
    for (int t = 0; t < nt; t++) free(tv[t]);
    free(tv);
    free(tn);
    free(tc);
    return ret;
}

/* histogram (codebook.py:23-27): bincount, symbol >= cap -> DataError. */
int orc_histogram(const uint32_t *sym, int64_t n, int64_t cap, int64_t *hist) {
    memset(hist, 0, (size_t)cap * sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) {
        if (sym[i] >= (uint64_t)cap) return ORC_E_DATA;
        hist[sym[i]]++;
    }
    return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * Huffman bit packing (huffman.py:46-61): concatenate the code words MSB
 * first; the final byte is zero padded.  Returns bit_len, or -1 when a symbol
 * has no code word (DataError), -2 if the output buffer is too small.
 * out must hold ceil(bit_len/8) bytes; it is fully written (zero padding).
 * ------------------------------------------------------------------------- */
int64_t orc_huff_encode(const uint32_t *sym, int64_t n, const uint8_t *lengths,
                        const uint64_t *codes, int64_t cap, uint8_t *out, int64_t out_cap) {
    uint64_t acc = 0; /* pending bits, right aligned */
    int nacc = 0;
    int64_t nbytes = 0, bits = 0;
    for (int64_t i = 0; i < n; i++) {
        uint32_t s = sym[i];
        if (s >= (uint64_t)cap || lengths[s] == 0) return -1;
        int L = lengths[s];
        uint64_t c = codes[s];
        bits += L;
        /* push L bits MSB first, in pieces so acc never exceeds 64 bits */
        while (L > 0) {
            int take = L > 32 ? 32 : L;
            uint64_t piece = (c >> (L - take)) & ((take == 64) ? ~0ull : ((1ull << take) - 1));
            acc = (acc << take) | piece;
            nacc += take;
            L -= take;
            while (nacc >= 8) {
                if (nbytes >= out_cap) return -2;
                out[nbytes++] = (uint8_t)(acc >> (nacc - 8));
                nacc -= 8;
            }
            acc &= (nacc ? ((1ull << nacc) - 1) : 0);
        }
    }
    if (nacc) {
        if (nbytes >= out_cap) return -2;
        out[nbytes++] = (uint8_t)(acc << (8 - nacc));
    }
    return bits;
}

/* ---------------------------------------------------------------------------
 * Canonical Huffman decode (huffman.py:64-122).  Tables per code length L:
 * first[L] = first canonical code of length L, cnt[L] = number of codes of
 * length L, off[L] = index of that first symbol in the (length, symbol)
 * sorted list `syms`.  The stream is walked bit by bit; a code word of length
 * L matches when first[L] <= acc < first[L] + cnt[L] (the reference's
 * limit[L] = first[L] + cnt[L]).
 * Returns the number of symbols emitted, or
 *   -1 code word longer than 64 bits, -2 more code words than `count`,
 *   -3 stream ends mid code word  (the reference's kernel status codes).
 * ------------------------------------------------------------------------- */
int64_t orc_huff_decode(const uint8_t *data, int64_t bit_len, int64_t count,
                        const uint64_t *first, const uint64_t *cnt, const int64_t *off,
                        const uint32_t *syms, uint32_t *out) {
    int64_t emitted = 0;
    uint64_t acc = 0;
    int len = 0;
    for (int64_t pos = 0; pos < bit_len; pos++) {
        uint64_t bit = (data[pos >> 3] >> (7 - (pos & 7))) & 1u;
        acc = (acc << 1) | bit;
        len++;
        if (len > 64) return -1;
        if (cnt[len] && acc >= first[len] && acc - first[len] < cnt[len]) {
            if (emitted == count) return -2;
            out[emitted++] = syms[off[len] + (int64_t)(acc - first[len])];
            acc = 0;
            len = 0;
        }
    }
    if (len != 0) return -3;
    return emitted;
}

/* ---------------------------------------------------------------------------
 * Run-length encode (rle.py:17-35): maximal runs; a run longer than max_run
 * (0xFFFFFFFF in the reference) is emitted as ceil(L/max_run) runs, all
 * max_run long except the last.  Returns the run count, or -1 if cap_runs is
 * too small.
 * ------------------------------------------------------------------------- */
int64_t orc_rle_encode(const uint32_t *sym, int64_t n, uint64_t max_run, uint32_t *values,
                       uint32_t *lengths, int64_t cap_runs) {
    int64_t r = 0;
    int64_t i = 0;
    while (i < n) {
        int64_t j = i + 1;
        while (j < n && sym[j] == sym[i]) j++;
        uint64_t L = (uint64_t)(j - i);
        while (L > 0) {
            uint64_t piece = L > max_run ? max_run : L;
            /* the reference splits as [MAX]*(reps-1) + [remainder] */
            uint64_t reps = (L + max_run - 1) / max_run;
            if (reps > 1) piece = max_run;
            if (r >= cap_runs) return -1;
            values[r] = sym[i];
            lengths[r] = (uint32_t)piece;
            r++;
            L -= piece;
        }
        i = j;
    }
    return r;
}

/* Run-length decode (rle.py:38-44).  Returns 0, or -1 on a zero-length run,
 * -2 if the runs do not sum to n. */
int orc_rle_decode(const uint32_t *values, const uint32_t *lengths, int64_t runs,
                   uint32_t *out, int64_t n) {
    int64_t total = 0;
    for (int64_t k = 0; k < runs; k++) {
        if (lengths[k] == 0) return -1;
        total += lengths[k];
    }
    if (total != n) return -2;
    int64_t pos = 0;
    for (int64_t k = 0; k < runs; k++)
        for (uint32_t t = 0; t < lengths[k]; t++) out[pos++] = values[k];
    return 0;
}

/* ---------------------------------------------------------------------------
 * Reconstruction from the chunk-major stream (reconstruct.py:22-88 +
 * pipeline.py:108-117): for each chunk, q' = code - r (+ outlier delta at the
 * outlier's position, fuse_outliers :22-32), overflow guard on the f64 sum of
 * |q'| (:48-53), inclusive prefix sums along x, then y, then z (:54-57), then
 * dequantize f64(code) * (2*eb_abs) cast to the output dtype (:79-88).
 *
 * out_pre (optional, may be NULL) receives the prequant integers in grid
 * order; out_vals (optional) the dequantized f32/f64 values in grid order.
 * Outliers must be sorted strictly by index (validated by the caller).
 * Returns 0, ORC_E_OVERFLOW, or ORC_E_DATA (non-finite dequantized value,
 * first offending offset in *bad_offset).
 * ------------------------------------------------------------------------- */
int orc_reconstruct_stream(const uint32_t *stream, int64_t nx, int64_t ny, int64_t nz, int ndim,
                           int64_t cx, int64_t cy, int64_t cz, int64_t radius,
                           const int64_t *out_idx, const int64_t *out_delta, int64_t n_out,
                           int64_t *out_pre, double eb_abs, int out_is_f64, void *out_vals,
                           int threads) {
    geom_t g = mkgeom(nx, ny, nz, cx, cy, cz);
    int64_t nchunks = g.nbx * g.nby * g.nbz;
    int64_t n = nx * ny * nz;
    /* fused deltas in grid order (fuse_outliers) */
    int64_t *fused = (int64_t *)malloc((size_t)n * sizeof(int64_t));
    if (!fused) return ORC_E_NOMEM;
    int overflow = 0;
    set_threads(threads);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t c = 0; c < nchunks; c++) {
        int64_t bx = c % g.nbx, by = (c / g.nbx) % g.nby, bz = c / (g.nbx * g.nby);
        int64_t x0 = bx * cx, y0 = by * cy, z0 = bz * cz;
        int64_t ex = cx < nx - x0 ? cx : nx - x0;
        int64_t ey = cy < ny - y0 ? cy : ny - y0;
        int64_t ez = cz < nz - z0 ? cz : nz - z0;
        int64_t pos = chunk_stream_base(&g, bx, by, bz);
        for (int64_t lz = 0; lz < ez; lz++)
            for (int64_t ly = 0; ly < ey; ly++)
                for (int64_t lx = 0; lx < ex; lx++, pos++)
                    fused[(x0 + lx) + nx * ((y0 + ly) + ny * (z0 + lz))] =
                        (int64_t)stream[pos] - radius;
    }
    for (int64_t k = 0; k < n_out; k++) fused[out_idx[k]] += out_delta[k];
#pragma omp parallel for schedule(dynamic, 64) reduction(| : overflow)
    for (int64_t c = 0; c < nchunks; c++) {
        int64_t bx = c % g.nbx, by = (c / g.nbx) % g.nby, bz = c / (g.nbx * g.nby);
        int64_t x0 = bx * cx, y0 = by * cy, z0 = bz * cz;
        int64_t ex = cx < nx - x0 ? cx : nx - x0;
        int64_t ey = cy < ny - y0 ? cy : ny - y0;
        int64_t ez = cz < nz - z0 ? cz : nz - z0;
#define AT(lx, ly, lz) fused[(x0 + (lx)) + nx * ((y0 + (ly)) + ny * (z0 + (lz)))]
        double tot = 0.0;
        for (int64_t lz = 0; lz < ez; lz++)
            for (int64_t ly = 0; ly < ey; ly++)
                for (int64_t lx = 0; lx < ex; lx++) {
                    int64_t v = AT(lx, ly, lz);
                    tot += fabs((double)v);
                }
        if (tot >= PSUM_LIMIT) { overflow = 1; continue; }
        for (int64_t lz = 0; lz < ez; lz++)
            for (int64_t ly = 0; ly < ey; ly++)
                for (int64_t lx = 1; lx < ex; lx++) AT(lx, ly, lz) += AT(lx - 1, ly, lz);
        if (ndim >= 2)
            for (int64_t lz = 0; lz < ez; lz++)
                for (int64_t ly = 1; ly < ey; ly++)
                    for (int64_t lx = 0; lx < ex; lx++) AT(lx, ly, lz) += AT(lx, ly - 1, lz);
        if (ndim >= 3)
            for (int64_t lz = 1; lz < ez; lz++)
                for (int64_t ly = 0; ly < ey; ly++)
                    for (int64_t lx = 0; lx < ex; lx++) AT(lx, ly, lz) += AT(lx, ly, lz - 1);
#undef AT
    }
    if (overflow) { free(fused); return ORC_E_OVERFLOW; }
    if (out_pre) memcpy(out_pre, fused, (size_t)n * sizeof(int64_t));
    int ret = ORC_OK;
    if (out_vals) {
        const double two_eb = 2.0 * eb_abs;
        if (out_is_f64) {
            double *o = (double *)out_vals;
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < n; i++) o[i] = (double)fused[i] * two_eb;
        } else {
            float *o = (float *)out_vals;
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < n; i++) o[i] = (float)((double)fused[i] * two_eb);
        }
    }
    free(fused);
    return ret;
}

/* First non-finite element (grid.py:176-180) and min/max; returns the
 * offending offset or -1. */
int64_t orc_finite_minmax(const void *vals, int is_f64, int64_t n, double *vmin, double *vmax) {
    double lo = INFINITY, hi = -INFINITY;
    for (int64_t i = 0; i < n; i++) {
        double v = is_f64 ? ((const double *)vals)[i] : (double)((const float *)vals)[i];
        if (!isfinite(v)) return i;
        if (v < lo) lo = v;
        if (v > hi) hi = v;
    }
    *vmin = lo;
    *vmax = hi;
    return -1;
}
