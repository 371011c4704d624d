// Interest-window codecs on device: notify::encode_delta
// and notify::decode_delta (notify.cpp:127-180), the wire form of a served or
// frozen interest delta (ServerCore::make_freeze, server.cpp:45-56).
//
// encode: varint(m_bits) || varint(ones) || varint(first set position) ||
//         varint(gap to the next set position) ... (LEB128, 7 bits per byte).
// A set-bit compaction with variable-length output, one filter word per thread:
// device-wide scans give every word (a) the last set position before it (the
// first gap's predecessor, a max-scan), (b) the popcount prefix (the header's
// count) and (c) its byte offset (a sum-scan of its varint lengths).
//
// decode: one 16-byte chunk per thread and the same scans over the byte stream
// (terminator bytes = bytes with the high bit clear; the varint ending at byte j
// starts after the previous terminator, found by a max-scan; the positions are a
// wrapping sum-scan of the gaps), with the reference's exact rejection rules: header varints
// present, 0 < m <= 2^32-1, a varint longer than 10 bytes or cut off by the end
// of the buffer, a zero gap after the first position, a position >= m (after the
// reference's wrapping uint64 addition), and a count that does not match the
// number of varints (trailing bytes) all make the result "nullopt".
#include <cuda_runtime.h>

#include <cstdint>
#include <cub/cub.cuh>

#include "scan.cuh"

namespace xpir {

namespace {

__device__ __forceinline__ uint32_t vlen(uint64_t v) {
    uint32_t n = 1;
    while (v >= 0x80) {
        v >>= 7;
        ++n;
    }
    return n;
}
__device__ __forceinline__ uint32_t vput(uint8_t* p, uint64_t v) {  // put_varint, notify.cpp:119-125
    uint32_t n = 0;
    while (v >= 0x80) {
        p[n++] = uint8_t(v) | 0x80;
        v >>= 7;
    }
    p[n++] = uint8_t(v);
    return n;
}
// get_varint (notify.cpp:127-137) over bytes [at, len): value, or false
__device__ __forceinline__ bool vget(const uint8_t* buf, uint64_t len, uint64_t& at, uint64_t& out) {
    uint64_t v = 0;
    int shift = 0;
    while (at < len && shift < 64) {
        const uint8_t b = buf[at++];
        v |= uint64_t(b & 0x7f) << shift;
        if (!(b & 0x80)) {
            out = v;
            return true;
        }
        shift += 7;
    }
    return false;
}

}  // namespace

// ---------------------------------------------------------------------------
// Grid-wide versions: one filter word (encode) / one 16-byte chunk (decode) per
// thread, with device-wide scans (CUB) between the passes.
// ---------------------------------------------------------------------------
namespace {

constexpr int DCH = 16;  // decode: body bytes per thread

__global__ void k_enc_a(const uint64_t* __restrict__ words, uint64_t nw, unsigned long long* __restrict__ pop,
                        unsigned long long* __restrict__ last1) {
    const uint64_t w = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (w >= nw) return;
    const uint64_t x = words[w];
    pop[w] = __popcll(x);
    last1[w] = x ? w * 64 + (63 - __clzll(x)) + 1 : 0;
}

__global__ void k_enc_b(const uint64_t* __restrict__ words, uint64_t nw, const unsigned long long* __restrict__ prev1,
                        unsigned long long* __restrict__ nbytes) {
    const uint64_t w = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (w >= nw) return;
    uint64_t x = words[w], prev = prev1[w];
    unsigned long long n = 0;
    while (x) {
        const uint64_t pos = w * 64 + (__ffsll(static_cast<long long>(x)) - 1);
        n += vlen(prev ? pos - (prev - 1) : pos);
        prev = pos + 1;
        x &= x - 1;
    }
    nbytes[w] = n;
}

// pop_ex / off_in are exclusive / inclusive scans; the header goes first
__global__ void k_enc_c(const uint64_t* __restrict__ words, uint64_t nw, uint32_t m_bits,
                        const unsigned long long* __restrict__ pop, const unsigned long long* __restrict__ pop_ex,
                        const unsigned long long* __restrict__ prev1, const unsigned long long* __restrict__ nbytes,
                        const unsigned long long* __restrict__ off_in, uint8_t* __restrict__ out, uint64_t cap,
                        unsigned long long* __restrict__ len_out) {
    const uint64_t w = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const unsigned long long ones = pop_ex[nw - 1] + pop[nw - 1];
    const uint64_t hdr = vlen(m_bits) + vlen(ones);
    const uint64_t total = hdr + off_in[nw - 1];
    if (w == 0) *len_out = total;
    if (w >= nw || total > cap || !out) return;
    if (w == 0) {
        const uint32_t n = vput(out, m_bits);
        vput(out + n, ones);
    }
    uint64_t x = words[w], prev = prev1[w];
    uint8_t* p = out + hdr + (off_in[w] - nbytes[w]);
    while (x) {
        const uint64_t pos = w * 64 + (__ffsll(static_cast<long long>(x)) - 1);
        p += vput(p, prev ? pos - (prev - 1) : pos);
        prev = pos + 1;
        x &= x - 1;
    }
}

// decode header (one thread): hdr[0] = verdict (0 ok, 1 malformed, 2 words too small),
// hdr[1] = m, hdr[2] = count, hdr[3] = body start, hdr[4] = header verdict (the
// later passes touch `words` only when the header was valid and fits)
__global__ void k_dec_hdr(const uint8_t* __restrict__ buf, uint64_t len, uint64_t words_cap,
                          unsigned long long* __restrict__ hdr) {
    uint64_t at = 0, m = 0, count = 0;
    int bad = 0;
    if (!vget(buf, len, at, m) || !vget(buf, len, at, count) || m == 0 || m > 0xffffffffull) bad = 1;
    else if ((m + 63) / 64 > words_cap) bad = 2;
    hdr[0] = bad;
    hdr[1] = m;
    hdr[2] = count;
    hdr[3] = bad ? len : at;
    hdr[4] = bad;
}

__global__ void k_dec_a(const uint8_t* __restrict__ buf, uint64_t len, const unsigned long long* __restrict__ hdr,
                        uint64_t nch, unsigned long long* __restrict__ nends, unsigned long long* __restrict__ lastend1) {
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= nch) return;
    const uint64_t at = hdr[3];
    const uint64_t b0 = max(at, t * DCH), b1 = min(len, (t + 1) * DCH);
    unsigned long long n = 0, l = 0;
    for (uint64_t j = b0; j < b1; ++j)
        if (!(buf[j] & 0x80)) {
            ++n;
            l = j + 1;
        }
    nends[t] = n;
    lastend1[t] = l;
}

__global__ void k_dec_b(const uint8_t* __restrict__ buf, uint64_t len, unsigned long long* __restrict__ hdr,
                        uint64_t nch, const unsigned long long* __restrict__ prevend1, unsigned long long* __restrict__ gsum) {
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= nch) return;
    const uint64_t at = hdr[3];
    const uint64_t b0 = max(at, t * DCH), b1 = min(len, (t + 1) * DCH);
    uint64_t start = prevend1[t] ? prevend1[t] : at;
    unsigned long long s = 0;
    for (uint64_t j = b0; j < b1; ++j) {
        if (buf[j] & 0x80) continue;
        uint64_t a = start, v = 0;
        if (j - start + 1 > 10 || !vget(buf, j + 1, a, v)) atomicExch(&hdr[0], 1ull);  // > 10 bytes (notify.cpp:130)
        s += v;
        start = j + 1;
    }
    gsum[t] = s;
}

__global__ void k_dec_c(const uint8_t* __restrict__ buf, uint64_t len, unsigned long long* __restrict__ hdr,
                        uint64_t nch, const unsigned long long* __restrict__ prevend1,
                        const unsigned long long* __restrict__ ends_ex, const unsigned long long* __restrict__ nends,
                        const unsigned long long* __restrict__ gbase, uint64_t* __restrict__ words) {
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= nch) return;
    if (hdr[4]) return;
    const uint64_t m = hdr[1], count = hdr[2], at = hdr[3];
    if (t == nch - 1) {  // exactly `count` varints, nothing after the last one (notify.cpp:166-178)
        const unsigned long long tot = ends_ex[t] + nends[t];
        if (tot != count || (len > at && (buf[len - 1] & 0x80))) atomicExch(&hdr[0], 1ull);
    }
    const uint64_t b0 = max(at, t * DCH), b1 = min(len, (t + 1) * DCH);
    uint64_t start = prevend1[t] ? prevend1[t] : at, pos = gbase[t], k = ends_ex[t];
    for (uint64_t j = b0; j < b1; ++j) {
        if (buf[j] & 0x80) continue;
        uint64_t a = start, v = 0;
        vget(buf, j + 1, a, v);
        if (k > 0 && v == 0) atomicExch(&hdr[0], 1ull);
        pos += v;
        if (pos >= m) atomicExch(&hdr[0], 1ull);
        else if (k < count) atomicOr(reinterpret_cast<unsigned long long*>(words) + (pos >> 6), 1ull << (pos & 63));
        start = j + 1;
        ++k;
    }
}

struct MaxU64 {
    __device__ __forceinline__ unsigned long long operator()(unsigned long long a, unsigned long long b) const {
        return a > b ? a : b;
    }
};

}  // namespace

size_t encode_delta_scratch_bytes(uint64_t nw) {
    size_t t1 = 0, t2 = 0;
    unsigned long long* p = nullptr;
    cub::DeviceScan::ExclusiveScan(nullptr, t1, p, p, MaxU64(), 0ull, int(nw));
    cub::DeviceScan::InclusiveSum(nullptr, t2, p, p, int(nw));
    return 6 * 8 * (nw + 1) + (t1 > t2 ? t1 : t2) + 256;
}

cudaError_t launch_encode_delta(const uint64_t* words, uint64_t nw, uint32_t m_bits, uint8_t* out, uint64_t cap,
                                unsigned long long* len_out, void* scratch, size_t scratch_bytes, cudaStream_t s) {
    if (nw == 0) return cudaErrorInvalidValue;
    auto* a = static_cast<unsigned long long*>(scratch);
    unsigned long long *pop = a, *last1 = a + nw, *prev1 = a + 2 * nw, *pop_ex = a + 3 * nw, *nb = a + 4 * nw,
                       *off = a + 5 * nw;
    void* tmp = a + 6 * (nw + 1);
    size_t tb = scratch_bytes - 6 * 8 * (nw + 1);
    const uint32_t g = uint32_t((nw + 255) / 256);
    k_enc_a<<<g, 256, 0, s>>>(words, nw, pop, last1);
    cudaError_t e = cub::DeviceScan::ExclusiveScan(tmp, tb, last1, prev1, MaxU64(), 0ull, int(nw), s);
    if (e != cudaSuccess) return e;
    tb = scratch_bytes - 6 * 8 * (nw + 1);
    e = cub::DeviceScan::ExclusiveSum(tmp, tb, pop, pop_ex, int(nw), s);
    if (e != cudaSuccess) return e;
    k_enc_b<<<g, 256, 0, s>>>(words, nw, prev1, nb);
    tb = scratch_bytes - 6 * 8 * (nw + 1);
    e = cub::DeviceScan::InclusiveSum(tmp, tb, nb, off, int(nw), s);
    if (e != cudaSuccess) return e;
    k_enc_c<<<g, 256, 0, s>>>(words, nw, m_bits, pop, pop_ex, prev1, nb, off, out, cap, len_out);
    count_launches(6);
    return cudaGetLastError();
}

size_t decode_delta_scratch_bytes(uint64_t len) {
    const uint64_t nch = (len + DCH - 1) / DCH + 1;
    size_t t1 = 0, t2 = 0;
    unsigned long long* p = nullptr;
    cub::DeviceScan::ExclusiveScan(nullptr, t1, p, p, MaxU64(), 0ull, int(nch));
    cub::DeviceScan::ExclusiveSum(nullptr, t2, p, p, int(nch));
    return 6 * 8 * (nch + 1) + (t1 > t2 ? t1 : t2) + 256;
}

// hdr: 5 x u64 (verdict in hdr[0], m in hdr[1] when done)
cudaError_t launch_decode_delta(const uint8_t* buf, uint64_t len, uint64_t* words, uint64_t words_cap,
                                unsigned long long* hdr, void* scratch, size_t scratch_bytes, cudaStream_t s) {
    const uint64_t nch = (len + DCH - 1) / DCH + 1;
    auto* a = static_cast<unsigned long long*>(scratch);
    unsigned long long *nends = a, *last1 = a + nch, *prev1 = a + 2 * nch, *ends_ex = a + 3 * nch, *gsum = a + 4 * nch,
                       *gbase = a + 5 * nch;
    void* tmp = a + 6 * (nch + 1);
    const size_t tb0 = scratch_bytes - 6 * 8 * (nch + 1);
    size_t tb = tb0;
    const uint32_t g = uint32_t((nch + 255) / 256);
    k_dec_hdr<<<1, 1, 0, s>>>(buf, len, words_cap, hdr);
    k_dec_a<<<g, 256, 0, s>>>(buf, len, hdr, nch, nends, last1);
    cudaError_t e = cub::DeviceScan::ExclusiveSum(tmp, tb, nends, ends_ex, int(nch), s);
    if (e != cudaSuccess) return e;
    tb = tb0;
    e = cub::DeviceScan::ExclusiveScan(tmp, tb, last1, prev1, MaxU64(), 0ull, int(nch), s);
    if (e != cudaSuccess) return e;
    k_dec_b<<<g, 256, 0, s>>>(buf, len, hdr, nch, prev1, gsum);
    tb = tb0;
    e = cub::DeviceScan::ExclusiveSum(tmp, tb, gsum, gbase, int(nch), s);
    if (e != cudaSuccess) return e;
    k_dec_c<<<g, 256, 0, s>>>(buf, len, hdr, nch, prev1, ends_ex, nends, gbase, words);
    count_launches(7);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// The write's interest field (wire.cpp:154-169): notify::encode_positions /
// decode_positions (notify.cpp:182-214), one thread per write. A field is
// varint(count) || varint(first) || varint(gaps) of the sorted positions,
// zero-padded to `cap` bytes (INTEREST_FIELD_LEN = 64 on the wire).

constexpr uint32_t POS_MAX_H = 128;

__global__ void k_encode_positions(const uint32_t* __restrict__ pos, uint32_t h, uint64_t n, uint32_t cap,
                                   uint8_t* __restrict__ out, uint8_t* __restrict__ ok) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t s[POS_MAX_H];
    for (uint32_t k = 0; k < h; ++k) {  // insertion sort (std::sort order, duplicates kept)
        const uint32_t v = pos[i * h + k];
        uint32_t j = k;
        while (j > 0 && s[j - 1] > v) {
            s[j] = s[j - 1];
            --j;
        }
        s[j] = v;
    }
    uint64_t need = vlen(h);
    for (uint32_t k = 0; k < h; ++k) need += vlen(k == 0 ? s[k] : s[k] - s[k - 1]);
    uint8_t* f = out + i * cap;
    uint32_t at = 0;
    if (need <= cap) {  // otherwise the reference throws: the field stays zero, ok = 0
        at = vput(f, h);
        for (uint32_t k = 0; k < h; ++k) at += vput(f + at, k == 0 ? s[k] : s[k] - s[k - 1]);
    }
    for (uint32_t k = at; k < cap; ++k) f[k] = 0;
    ok[i] = need <= cap ? 1 : 0;
}

__global__ void k_decode_positions(const uint8_t* __restrict__ fields, uint32_t cap, uint64_t n,
                                   uint32_t* __restrict__ pos, uint32_t* __restrict__ count) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint8_t* f = fields + i * cap;
    uint32_t* o = pos + i * cap;
    uint64_t at = 0, c = 0, p = 0;
    uint32_t res = 0xffffffffu;  // std::nullopt
    if (vget(f, cap, at, c) && c <= uint64_t(cap) * 8) {
        uint64_t k = 0;
        for (; k < c; ++k) {
            uint64_t gap;
            if (!vget(f, cap, at, gap)) break;
            p = k == 0 ? gap : p + gap;  // uint64 arithmetic, wrapping as the reference's
            if (p > 0xffffffffull) break;
            if (k < cap) o[k] = uint32_t(p);  // a parsed varint takes >= 1 byte: k < cap
        }
        if (k == c) res = uint32_t(c);
    }
    count[i] = res;
}

cudaError_t launch_encode_positions(const uint32_t* pos, uint32_t h, uint64_t n, uint32_t cap, uint8_t* out,
                                    uint8_t* ok, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_encode_positions<<<uint32_t((n + 127) / 128), 128, 0, s>>>(pos, h, n, cap, out, ok);
    return cudaGetLastError();
}

cudaError_t launch_decode_positions(const uint8_t* fields, uint32_t cap, uint64_t n, uint32_t* pos, uint32_t* count,
                                    cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_decode_positions<<<uint32_t((n + 127) / 128), 128, 0, s>>>(fields, cap, n, pos, count);
    return cudaGetLastError();
}

}  // namespace xpir
