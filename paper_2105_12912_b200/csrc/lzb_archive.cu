// Device-side assembly of a Huffman archive (single-sync compress).
//
// Archive layout (P/pipeline.py:184-221, the same bytes compress() writes):
//   [0, 130)            header "<8sHBB3I3IBdddIBQQ6Q" (P/pipeline.py:184-194)
//   [130, 136)          zero
//   [136, 136 + cap)    code lengths (the code book section)
//   ... zero ...        up to sym_off = align8(136 + cap)
//   [sym_off, +16)      <QQ> bit_len, count
//   [sym_off + 16, +nb) the bit stream (lzb_huff_encode writes it in place)
//   ... zero ...        up to out_off = align8(sym_off + 16 + nb)
//   [out_off, +16 n_out) outlier records
//
// The host knows everything but nb (from the device code book) and n_out
// (from K1): it passes the header with those fields unset and this kernel
// patches outlier_count, sym_len, out_off and out_len, so the whole compress
// runs without a mid-pipeline read-back.
#include "lzb_common.cuh"

namespace lzb {

struct ArcHeader {
    uint8_t b[136];
};

// byte offsets of the patched fields in the packed header
constexpr uint32_t kHdrOutCount = 74, kHdrSymLen = 106, kHdrOutOff = 114, kHdrOutLen = 122;
constexpr uint32_t kHdrBytes = 130, kSectionBase = 136;

__device__ __forceinline__ void put_u64(uint8_t *dst, uint64_t v) {
#pragma unroll
    for (int i = 0; i < 8; i++) dst[i] = (uint8_t)(v >> (8 * i));
}

__global__ void __launch_bounds__(256) k_archive_finalize(uint8_t *arc, uint64_t arc_bytes, ArcHeader h,
                                                         uint64_t sym_off, const uint8_t *lengths, uint32_t cap,
                                                         const lzb_dstatus *st_q, const lzb_dstatus *st_b,
                                                         const uint2 *records, lzb_dstatus *st) {
    if (st_q->code != 0 || st_b->code != 0) return;  // the host reports those
    const uint64_t bits = st_b->u[0], count = st_b->u[1], n_out = st_q->u[0];
    const uint64_t nb = (bits + 7) / 8;
    const uint64_t sym_len = 16 + nb;
    const uint64_t out_off = (sym_off + sym_len + 7) & ~7ull;
    const uint64_t total = out_off + 16 * n_out;
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
    if (tid == 0) {
        st->u[0] = total;
        st->u[1] = out_off;
        if (total > arc_bytes) set_status(st, LZB_E_CAPACITY);
    }
    if (total > arc_bytes) return;
    if (blockIdx.x == 0) {
        for (uint32_t i = threadIdx.x; i < kSectionBase; i += blockDim.x) {
            uint8_t v = i < kHdrBytes ? h.b[i] : 0;
            if (i >= kHdrOutCount && i < kHdrOutCount + 8) v = (uint8_t)(n_out >> (8 * (i - kHdrOutCount)));
            if (i >= kHdrSymLen && i < kHdrSymLen + 8) v = (uint8_t)(sym_len >> (8 * (i - kHdrSymLen)));
            if (i >= kHdrOutOff && i < kHdrOutOff + 8) v = (uint8_t)(out_off >> (8 * (i - kHdrOutOff)));
            if (i >= kHdrOutLen && i < kHdrOutLen + 8) v = (uint8_t)((16 * n_out) >> (8 * (i - kHdrOutLen)));
            arc[i] = v;
        }
        for (uint32_t i = threadIdx.x; i < (uint32_t)(sym_off - kSectionBase); i += blockDim.x)
            arc[kSectionBase + i] = i < cap ? lengths[i] : 0;
        if (threadIdx.x == 0) {
            put_u64(arc + sym_off, bits);
            put_u64(arc + sym_off + 8, count);
        }
        for (uint64_t i = sym_off + sym_len + threadIdx.x; i < out_off; i += blockDim.x) arc[i] = 0;
    }
    uint2 *dst = reinterpret_cast<uint2 *>(arc + out_off);  // out_off is 8-aligned, arc 256-aligned
    for (uint64_t i = tid; i < 2 * n_out; i += nthr) dst[i] = records[i];
}

}  // namespace lzb

using namespace lzb;

static int sm_count() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    return sms;
}

extern "C" int lzb_archive_finalize_huff(uint8_t *arc, uint64_t arc_bytes, const uint8_t *header,
                                         uint64_t sym_off, const uint8_t *lengths, uint32_t cap,
                                         const lzb_dstatus *st_quant, const lzb_dstatus *st_book,
                                         const void *records, lzb_dstatus *st, void *stream) {
    if (!arc || !header || !lengths || !st_quant || !st_book || !st || cap == 0 ||
        sym_off < kSectionBase + cap || (sym_off & 7) || (reinterpret_cast<uintptr_t>(arc) & 7) ||
        (reinterpret_cast<uintptr_t>(records) & 7))
        return LZB_E_ARG;
    cudaStream_t s = as_stream(stream);
    ArcHeader h;
    for (uint32_t i = 0; i < kSectionBase; i++) h.b[i] = i < kHdrBytes ? header[i] : 0;
    LZB_CUDA_TRY(cudaMemsetAsync(st, 0, sizeof(lzb_dstatus), s));
    const int sms = sm_count();
    k_archive_finalize<<<(unsigned)(sms > 0 ? sms : 1), 256, 0, s>>>(arc, arc_bytes, h, sym_off, lengths, cap,
                                                                    st_quant, st_book,
                                                                    static_cast<const uint2 *>(records), st);
    LZB_LAUNCH_CHECK();
    return LZB_OK;
}
