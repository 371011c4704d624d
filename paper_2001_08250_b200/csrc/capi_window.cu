// C-ABI (include/xpir.h): the interest window and its codecs — notify::Window (notify.cpp:54-180).
#include "capi_internal.cuh"

// ===========================================================================
// interest window
// ===========================================================================
// Per-device grow-only scratch + stream for the standalone codec entry points.
struct CodecScratch {
    std::mutex mu;
    DevBuf buf;
    cudaStream_t stream = nullptr;
    unsigned long long* host = nullptr;  // pinned, 2 words
};
static CodecScratch& codec_scratch(int device) {
    static std::mutex m;
    static CodecScratch* per[64] = {};
    std::lock_guard<std::mutex> lk(m);
    const int d = device >= 0 && device < 64 ? device : 0;
    if (!per[d]) {  // intentionally leaked (no teardown after the CUDA runtime)
        per[d] = new CodecScratch;
        cudaStreamCreateWithFlags(&per[d]->stream, cudaStreamNonBlocking);
        cudaHostAlloc(reinterpret_cast<void**>(&per[d]->host), 16, cudaHostAllocPortable);
    }
    return *per[d];
}


extern "C" {

int xpir_window_create(int device, uint32_t m_bits, uint32_t h, uint32_t w, xpir_window** out) {
    if (!out) return fail(XPIR_EINVAL, "window_create: null out");
    if (w == 0) return fail(XPIR_EINVAL, "Window: need at least one delta");   // notify.cpp:55
    if (m_bits == 0 || h == 0) return fail(XPIR_EINVAL, "Window: bad bloom params");  // :56
    int ndev = 0;
    XCK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(XPIR_EINVAL, "window_create: bad device");
    DeviceGuard g(device);
    auto* win = new xpir_window;
    win->device = device;
    win->m = m_bits;
    win->h = h;
    win->w = w;
    win->words = (uint64_t(m_bits) + 63) / 64;
    unsigned long long* d = nullptr;
    cudaError_t e = cudaMalloc(&d, 8 * win->words);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&win->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMemsetAsync(d, 0, 8 * win->words, win->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(win->stream);
    if (e == cudaSuccess) e = win->stage.ensure(4096);  // pinned position staging (absorb)
    if (e != cudaSuccess) {
        if (d) cudaFree(d);
        delete win;
        return fail(XPIR_ECUDA, cudaGetErrorString(e));
    }
    win->deltas.push_back(d);
    *out = win;
    return XPIR_OK;
}

int xpir_window_destroy(xpir_window* win) {
    if (!win) return XPIR_OK;
    DeviceGuard g(win->device);
    cudaStreamSynchronize(win->stream);
    for (auto* d : win->deltas) cudaFree(d);
    win->pos.release();
    win->seqs.release();
    win->scratch.release();
    win->enc.release();
    win->stage.release();
    win->dstage.release();
    cudaStreamDestroy(win->stream);
    delete win;
    return XPIR_OK;
}

int xpir_window_absorb_dev(xpir_window* win, const uint32_t* d_pos, uint64_t n, void* stream) {
    if (!win) return fail(XPIR_EINVAL, "window_absorb: null window");
    if (!n) return XPIR_OK;
    if (!d_pos) return fail(XPIR_EINVAL, "window_absorb: null buffer");
    DeviceGuard g(win->device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : win->stream;
    XCK(win->scratch.ensure(16));
    XCK(launch_absorb(d_pos, n, win->m, win->deltas.back(), win->scratch.as<unsigned long long>(), s));
    count_launches(2);
    unsigned long long first_bad = 0;
    XCK(cudaMemcpyAsync(&first_bad, win->scratch.p, 8, cudaMemcpyDeviceToHost, s));
    XCK(cudaStreamSynchronize(s));
    if (first_bad != ~0ull) return fail(XPIR_EINVAL, "Window: position out of range");
    return XPIR_OK;
}

int xpir_window_absorb(xpir_window* win, const uint32_t* pos, uint64_t n) {
    if (!win) return fail(XPIR_EINVAL, "window_absorb: null window");
    if (!n) return XPIR_OK;
    if (!pos) return fail(XPIR_EINVAL, "window_absorb: null buffer");
    std::lock_guard<std::mutex> lk(win->mu);
    DeviceGuard g(win->device);
    XCK(win->pos.ensure(4 * n));
    XCK(cudaMemcpyAsync(win->pos.p, pos, 4 * n, cudaMemcpyHostToDevice, win->stream));
    return xpir_window_absorb_dev(win, win->pos.as<uint32_t>(), n, win->stream);
}

}  // extern "C"

int window_absorb_prechecked(xpir_window* win, const uint32_t* pos, uint64_t n) {
    if (!n) return XPIR_OK;
    std::lock_guard<std::mutex> lk(win->mu);
    DeviceGuard g(win->device);
    XCK(win->stage.ensure(4 * n));
    std::memcpy(win->stage.p, pos, 4 * n);
    XCK(win->pos.ensure(4 * n));
    XCK(cudaMemcpyAsync(win->pos.p, win->stage.p, 4 * n, cudaMemcpyHostToDevice, win->stream));
    XCK(win->stage.release_after(win->stream));
    XCK(launch_absorb_unchecked(win->pos.as<uint32_t>(), n, win->deltas.back(), win->stream));
    count_launches(1);
    return XPIR_OK;
}

extern "C" {

int xpir_window_absorb_interest(xpir_window* win, const uint8_t id[16], const uint64_t* seqs,
                                uint64_t n) {
    if (!win || !id) return fail(XPIR_EINVAL, "window_absorb_interest: null argument");
    if (!n) return XPIR_OK;
    if (!seqs) return fail(XPIR_EINVAL, "window_absorb_interest: null buffer");
    std::lock_guard<std::mutex> lk(win->mu);
    DeviceGuard g(win->device);
    XCK(win->seqs.ensure(8 * n));
    XCK(cudaMemcpyAsync(win->seqs.p, seqs, 8 * n, cudaMemcpyHostToDevice, win->stream));
    XCK(launch_interest(id, win->seqs.as<uint64_t>(), n, win->h, win->m, nullptr, win->deltas.back(),
                        win->stream));
    count_launches(1);
    XCK(cudaStreamSynchronize(win->stream));
    return XPIR_OK;
}

int xpir_window_absorb_interest_dev(xpir_window* win, const uint8_t id[16], const uint64_t* d_seqs, uint64_t n,
                                    void* stream) {
    if (!win || !id) return fail(XPIR_EINVAL, "window_absorb_interest: null argument");
    if (!n) return XPIR_OK;
    if (!d_seqs) return fail(XPIR_EINVAL, "window_absorb_interest: null buffer");
    DeviceGuard g(win->device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : win->stream;
    XCK(launch_interest(id, d_seqs, n, win->h, win->m, nullptr, win->deltas.back(), s));
    count_launches(1);
    return XPIR_OK;
}

int xpir_window_rotate(xpir_window* win) {  // notify.cpp:67-73
    if (!win) return fail(XPIR_EINVAL, "window_rotate: null window");
    std::lock_guard<std::mutex> lk(win->mu);
    DeviceGuard g(win->device);
    // push an empty delta, pop from the front while size > W: at capacity the
    // popped delta's buffer is recycled (zeroed in stream order) instead of a
    // cudaMalloc + cudaFree per rotation
    unsigned long long* d = nullptr;
    if (!win->deltas.empty() && win->deltas.size() >= win->w) {
        d = win->deltas.front();
        win->deltas.pop_front();
        win->base++;
    } else {
        XCK(cudaMalloc(&d, 8 * win->words));
    }
    XCK(cudaMemsetAsync(d, 0, 8 * win->words, win->stream));
    // absorbs may come on the caller's stream: the new delta is zero before any of them
    XCK(cudaStreamSynchronize(win->stream));
    win->deltas.push_back(d);
    return XPIR_OK;
}

int xpir_window_info(const xpir_window* win, uint64_t* size, uint64_t* base) {
    if (!win) return fail(XPIR_EINVAL, "window_info: null window");
    if (size) *size = win->deltas.size();
    if (base) *base = win->base;
    return XPIR_OK;
}

int xpir_window_delta(const xpir_window* win, uint64_t i, uint64_t* out) {
    if (!win || !out) return fail(XPIR_EINVAL, "window_delta: null argument");
    if (i >= win->deltas.size()) return fail(XPIR_EINVAL, "window_delta: index out of range");
    DeviceGuard g(win->device);
    XCK(cudaStreamSynchronize(win->stream));
    XCK(cudaMemcpy(out, win->deltas[i], 8 * win->words, cudaMemcpyDeviceToHost));
    return XPIR_OK;
}

int xpir_window_digest(const xpir_window* win, uint8_t out[32]) {  // notify.cpp:90-107
    if (!win) return fail(XPIR_EINVAL, "window_digest: null argument");
    return xpir_window_digest_n(win, win->deltas.size(), out);
}

int xpir_window_digest_n(const xpir_window* win, uint64_t count, uint8_t out[32]) {  // Window::digest(count)
    if (!win || !out) return fail(XPIR_EINVAL, "window_digest: null argument");
    if (count > win->deltas.size()) return fail(XPIR_EINVAL, "Window::digest: count too large");  // notify.cpp:92
    // every delta in one batch of async copies into pinned memory, one sync (a
    // freeze digests the whole window: round 1 paid a sync + copy per delta)
    std::lock_guard<std::mutex> lk(win->mu);
    DeviceGuard g(win->device);
    const size_t row = 8 * win->words;
    XCK(win->dstage.ensure(count ? row * count : 1));
    for (uint64_t i = 0; i < count; ++i)
        XCK(cudaMemcpyAsync(win->dstage.p + i * row, win->deltas[i], row, cudaMemcpyDeviceToHost, win->stream));
    XCK(win->dstage.release_after(win->stream));
    XCK(cudaStreamSynchronize(win->stream));
    HostBlake2b h(32);
    const char* tag = "interest-window-v1";
    h.update(reinterpret_cast<const uint8_t*>(tag), std::strlen(tag));
    h.update_u64be(win->m);
    h.update_u64be(win->h);
    h.update_u64be(win->w);
    h.update_u64be(win->base);
    h.update_u64be(count);
    for (uint64_t i = 0; i < count; ++i) h.update(win->dstage.p + i * row, row);  // LE words
    h.final(out);
    return XPIR_OK;
}

// notify::encode_delta (notify.cpp:139-157) of delta i (0 = oldest) on device.
// out == NULL: size query. Otherwise out must hold *len bytes (EINVAL if cap is short).
int xpir_window_encode_delta(xpir_window* win, uint64_t i, uint8_t* out, uint64_t cap, uint64_t* len) {
    if (!win || !len) return fail(XPIR_EINVAL, "window_encode_delta: null argument");
    std::lock_guard<std::mutex> lk(win->mu);
    if (i >= win->deltas.size()) return fail(XPIR_EINVAL, "window_encode_delta: no such delta");
    DeviceGuard g(win->device);
    cudaStream_t s = win->stream;
    // worst case: every bit set, 5-byte varints
    const uint64_t worst = 20 + 5ull * 64 * win->words;
    const size_t sb = encode_delta_scratch_bytes(win->words);
    XCK(win->enc.ensure(16 + sb + worst));
    unsigned long long* dlen = win->enc.as<unsigned long long>();  // 8-byte aligned head
    void* scratch = win->enc.as<uint8_t>() + 16;
    uint8_t* denc = win->enc.as<uint8_t>() + 16 + sb;
    XCK(launch_encode_delta(reinterpret_cast<const uint64_t*>(win->deltas[i]), win->words, win->m, denc, worst,
                            dlen, scratch, sb, s));
    unsigned long long n = 0;
    XCK(cudaMemcpyAsync(&n, dlen, 8, cudaMemcpyDeviceToHost, s));
    XCK(cudaStreamSynchronize(s));
    *len = n;
    if (!out) return XPIR_OK;
    if (cap < n) return fail(XPIR_EINVAL, "window_encode_delta: output buffer too small");
    XCK(cudaMemcpyAsync(out, denc, n, cudaMemcpyDeviceToHost, s));
    XCK(cudaStreamSynchronize(s));
    return XPIR_OK;
}

// Device buffers: d_words (ceil(m/64) words) -> d_out (cap bytes); *len = encoded size.
int xpir_encode_delta_dev(int device, const uint64_t* d_words, uint32_t m_bits, uint8_t* d_out, uint64_t cap,
                          uint64_t* len, void* stream) {
    if (!d_words || !len || m_bits == 0) return fail(XPIR_EINVAL, "encode_delta: bad argument");
    DeviceGuard g(device);
    CodecScratch& cs = codec_scratch(device);
    std::lock_guard<std::mutex> lk(cs.mu);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : cs.stream;
    const uint64_t nw = (uint64_t(m_bits) + 63) / 64;
    const size_t sb = encode_delta_scratch_bytes(nw);
    XCK(cs.buf.ensure(16 + sb));
    unsigned long long* dlen = cs.buf.as<unsigned long long>();
    XCK(launch_encode_delta(d_words, nw, m_bits, d_out, d_out ? cap : 0, dlen, cs.buf.as<uint8_t>() + 16, sb, s));
    XCK(cudaMemcpyAsync(cs.host, dlen, 8, cudaMemcpyDeviceToHost, s));
    XCK(cudaStreamSynchronize(s));
    const unsigned long long n = cs.host[0];
    *len = n;
    if (d_out && cap < n) return fail(XPIR_EINVAL, "encode_delta: output buffer too small");
    return XPIR_OK;
}

// notify::encode_positions (notify.cpp:182-196) for n writes of h positions each
// into cap-byte fields; d_ok[i] = 0 where the reference throws (too long).
int xpir_encode_positions_dev(int device, const uint32_t* d_pos, uint32_t h, uint64_t n, uint32_t cap,
                              uint8_t* d_fields, uint8_t* d_ok, void* stream) {
    if (n && (!d_fields || !d_ok || (h && !d_pos))) return fail(XPIR_EINVAL, "encode_positions: null buffer");
    if (h > 128 || cap == 0 || cap > 4096) return fail(XPIR_EINVAL, "encode_positions: h <= 128, 1 <= cap <= 4096");
    DeviceGuard g(device);
    XCK(launch_encode_positions(d_pos, h, n, cap, d_fields, d_ok, static_cast<cudaStream_t>(stream)));
    count_launches(1);
    if (!stream) XCK(cudaStreamSynchronize(nullptr));
    return XPIR_OK;
}

// notify::decode_positions (notify.cpp:198-214) of n cap-byte fields: d_count[i] =
// the count (positions in d_pos[i*cap ..]) or 0xffffffff for std::nullopt.
int xpir_decode_positions_dev(int device, const uint8_t* d_fields, uint32_t cap, uint64_t n, uint32_t* d_pos,
                              uint32_t* d_count, void* stream) {
    if (n && (!d_fields || !d_pos || !d_count)) return fail(XPIR_EINVAL, "decode_positions: null buffer");
    if (cap == 0 || cap > 4096) return fail(XPIR_EINVAL, "decode_positions: 1 <= cap <= 4096");
    DeviceGuard g(device);
    XCK(launch_decode_positions(d_fields, cap, n, d_pos, d_count, static_cast<cudaStream_t>(stream)));
    count_launches(1);
    if (!stream) XCK(cudaStreamSynchronize(nullptr));
    return XPIR_OK;
}

// notify::decode_delta (notify.cpp:139-180). EINVAL = the reference's nullopt.
// words == NULL: header only (*m_bits). Otherwise words must hold ceil(m/64).
int xpir_decode_delta(int device, const uint8_t* buf, uint64_t len, uint32_t* m_bits, uint64_t* words,
                      uint64_t words_cap) {
    if (!m_bits || (len && !buf)) return fail(XPIR_EINVAL, "decode_delta: null argument");
    DeviceGuard g(device);
    CodecScratch& cs = codec_scratch(device);
    std::lock_guard<std::mutex> lk(cs.mu);
    cudaStream_t s = cs.stream;
    const uint64_t cap_words = words ? words_cap : 0;
    const size_t sb = decode_delta_scratch_bytes(len);
    const uint64_t wbytes = 8 * (cap_words ? cap_words : 1);
    const uint64_t o_scr = 64, o_buf = 64 + ((sb + 255) & ~size_t(255)), o_words = o_buf + ((len + 16 + 255) & ~uint64_t(255));
    XCK(cs.buf.ensure(o_words + wbytes));
    uint8_t* base = cs.buf.as<uint8_t>();
    unsigned long long* dres = cs.buf.as<unsigned long long>();
    uint64_t* dwords = reinterpret_cast<uint64_t*>(base + o_words);
    if (len) XCK(cudaMemcpyAsync(base + o_buf, buf, len, cudaMemcpyHostToDevice, s));
    XCK(cudaMemsetAsync(dwords, 0, wbytes, s));
    XCK(launch_decode_delta(base + o_buf, len, dwords, cap_words, dres, base + o_scr, sb, s));
    XCK(cudaMemcpyAsync(cs.host, dres, 16, cudaMemcpyDeviceToHost, s));
    XCK(cudaStreamSynchronize(s));
    const unsigned long long verdict = cs.host[0], m = cs.host[1];
    if (verdict == 1) return fail(XPIR_EINVAL, "decode_delta: malformed delta");
    *m_bits = uint32_t(m);
    if (verdict == 2) {
        if (!words) return XPIR_OK;  // header query
        return fail(XPIR_EINVAL, "decode_delta: words buffer too small");
    }
    XCK(cudaMemcpyAsync(words, dwords, 8 * ((m + 63) / 64), cudaMemcpyDeviceToHost, s));
    XCK(cudaStreamSynchronize(s));
    return XPIR_OK;
}

}  // extern "C"

