// extern "C" boundary (include/xpir.h) over the sm_100a kernels in scan.cu and
// write.cu. Host-side bookkeeping only: argument validation with the
// reference's error conditions, device memory ownership, kernel dispatch.
// There is no CPU compute path: every answer, table mutation and filter update
// is produced by a kernel, and the library fails (XPIR_ECUDA) without a GPU.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/xpir.h"
#include "prims.cuh"
#include "scan.cuh"

namespace xpir {
static std::atomic<uint64_t> g_launches{0};
void count_launches(uint64_t n) { g_launches += n; }
int set_error(int code, const std::string& msg);
}  // namespace xpir

using namespace xpir;

namespace {

thread_local std::string g_err;
std::atomic<int> g_last_kernel{0};
xpir_scan_opts g_opts{};
std::mutex g_opts_mu;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

}  // namespace

int xpir::set_error(int code, const std::string& msg) { return fail(code, msg); }

namespace {

#define XCK(expr)                                                                       \
    do {                                                                                \
        cudaError_t e_ = (expr);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return fail(XPIR_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

int num_sms(int dev) {
    static int cache[64] = {0};
    if (dev >= 0 && dev < 64 && cache[dev]) return cache[dev];
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (dev >= 0 && dev < 64) cache[dev] = n;
    return n;
}

// Grow-only device scratch buffer.
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t n) {
        if (n <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t want = std::max(n, size_t(256));
        cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

uint64_t round16(uint64_t x) { return (x + 15) & ~uint64_t(15); }

// Host BLAKE2b (same algorithm as the device port in prims.cuh), incremental,
// used for the digests that the reference computes over whole tables/windows.
struct HostBlake2b {
    uint64_t h[8];
    uint64_t t = 0;
    uint8_t buf[128];
    size_t buflen = 0, outlen;
    explicit HostBlake2b(size_t out) : outlen(out) {
        for (int i = 0; i < 8; ++i) h[i] = b2_iv(i);
        h[0] ^= 0x01010000ULL ^ out;
    }
    void block(bool last) {
        uint64_t m[16];
        for (int i = 0; i < 16; ++i) m[i] = ld64le(buf + 8 * i);
        blake2b_compress(h, m, t, 0, last);
    }
    void update(const uint8_t* in, size_t len) {
        while (len) {
            if (buflen == 128) {
                t += 128;
                block(false);
                buflen = 0;
            }
            size_t take = std::min(len, 128 - buflen);
            std::memcpy(buf + buflen, in, take);
            buflen += take;
            in += take;
            len -= take;
        }
    }
    void update_u64be(uint64_t v) {
        uint8_t b[8];
        for (int i = 0; i < 8; ++i) b[i] = uint8_t(v >> (56 - 8 * i));
        update(b, 8);
    }
    void final(uint8_t* out) {
        t += buflen;
        std::memset(buf + buflen, 0, 128 - buflen);
        block(true);
        uint8_t full[64];
        for (int i = 0; i < 8; ++i)
            for (int k = 0; k < 8; ++k) full[8 * i + k] = uint8_t(h[i] >> (8 * k));
        std::memcpy(out, full, outlen);
    }
};

}  // namespace

// ===========================================================================
// store
// ===========================================================================
struct xpir_store {
    int device;
    uint32_t N, S, lo, hi;
    uint64_t epoch = 0;
    uint8_t* data = nullptr;
    cudaStream_t stream = nullptr;
    DevBuf q, out, seeds, masks, qwin, qx, idx;
    std::mutex mu;
    // Query-window scratch of the device-pointer entry points, one per caller
    // stream, so calls on different streams may run concurrently (read batcher).
    std::mutex scratch_mu;
    std::vector<std::pair<cudaStream_t, DevBuf*>> qwin_by_stream;
    DevBuf& qwin_for(cudaStream_t s) {
        if (s == stream) return qwin;
        std::lock_guard<std::mutex> lk(scratch_mu);
        for (auto& e : qwin_by_stream)
            if (e.first == s) return *e.second;
        qwin_by_stream.emplace_back(s, new DevBuf);
        return *qwin_by_stream.back().second;
    }
    uint32_t nb() const { return hi - lo; }
    uint64_t bytes() const { return uint64_t(nb()) * S; }
    uint64_t byte_lo() const { return lo / 8; }
    uint64_t nbytes_window() const { return (uint64_t(hi) + 7) / 8 - lo / 8; }
};

extern "C" {

const char* xpir_last_error(void) { return g_err.c_str(); }
int xpir_version(void) { return 1; }
uint64_t xpir_launch_count(void) { return g_launches.load(); }

int xpir_set_scan_opts(const xpir_scan_opts* o) {
    std::lock_guard<std::mutex> lk(g_opts_mu);
    g_opts = o ? *o : xpir_scan_opts{};
    return XPIR_OK;
}
int xpir_last_scan_kernel(void) { return g_last_kernel.load(); }

}  // extern "C"

// Scan-kernel event timing (bench.py's roofline.achieved denominator).
namespace {
std::mutex g_tmu;
bool g_timing = false;
std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_events;

void timing_begin(cudaStream_t s, cudaEvent_t* a) {
    *a = nullptr;
    std::lock_guard<std::mutex> lk(g_tmu);
    if (!g_timing) return;
    cudaEventCreate(a);
    cudaEventRecord(*a, s);
}
void timing_end(cudaStream_t s, cudaEvent_t a) {
    if (!a) return;
    cudaEvent_t b;
    cudaEventCreate(&b);
    cudaEventRecord(b, s);
    std::lock_guard<std::mutex> lk(g_tmu);
    g_events.emplace_back(a, b);
}
}  // namespace

extern "C" {

int xpir_scan_timing(int enable) {
    std::lock_guard<std::mutex> lk(g_tmu);
    g_timing = enable != 0;
    return XPIR_OK;
}

int xpir_scan_timing_collect(double* total_ms, uint32_t* launches) {
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
    {
        std::lock_guard<std::mutex> lk(g_tmu);
        ev.swap(g_events);
    }
    double tot = 0;
    for (auto& p : ev) {
        float ms = 0;
        XCK(cudaEventSynchronize(p.second));
        XCK(cudaEventElapsedTime(&ms, p.first, p.second));
        tot += ms;
        cudaEventDestroy(p.first);
        cudaEventDestroy(p.second);
    }
    if (total_ms) *total_ms = tot;
    if (launches) *launches = uint32_t(ev.size());
    return XPIR_OK;
}

int xpir_measure_peaks(int device, double* lop3_per_s, double* smem_bps, double* sm_clock_mhz) {
    DeviceGuard g(device);
    cudaStream_t s;
    XCK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaError_t e = run_peak_kernels(num_sms(device), lop3_per_s, smem_bps, s);
    count_launches(4);
    cudaStreamDestroy(s);
    XCK(e);
    if (sm_clock_mhz) {
        int khz = 0;
        cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, device);
        *sm_clock_mhz = khz / 1000.0;
    }
    return XPIR_OK;
}

int xpir_probe_tmem(int device, int variant, double* bytes_per_clk_sm) {
    DeviceGuard g(device);
    XCK(run_tmem_probe(variant, num_sms(device), bytes_per_clk_sm));
    XCK(cudaDeviceSynchronize());
    count_launches(2);
    return XPIR_OK;
}

int xpir_dev_alloc(int device, uint64_t bytes, void** d_ptr) {
    if (!d_ptr) return fail(XPIR_EINVAL, "dev_alloc: null out");
    DeviceGuard g(device);
    cudaError_t e = cudaMalloc(d_ptr, std::max<uint64_t>(bytes, 16));
    if (e != cudaSuccess) return fail(XPIR_ENOMEM, std::string("dev_alloc: ") + cudaGetErrorString(e));
    return XPIR_OK;
}

int xpir_dev_free(int device, void* d_ptr) {
    DeviceGuard g(device);
    XCK(cudaFree(d_ptr));
    return XPIR_OK;
}

int xpir_ipc_get_handle(int device, const void* d_ptr, uint8_t handle[64]) {
    if (!d_ptr || !handle) return fail(XPIR_EINVAL, "ipc_get_handle: null argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    DeviceGuard g(device);
    cudaIpcMemHandle_t h;
    XCK(cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr)));
    std::memcpy(handle, &h, 64);
    return XPIR_OK;
}

int xpir_ipc_open(int device, const uint8_t handle[64], void** d_ptr) {
    if (!handle || !d_ptr) return fail(XPIR_EINVAL, "ipc_open: null argument");
    DeviceGuard g(device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    XCK(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return XPIR_OK;
}

int xpir_ipc_close(int device, void* d_ptr) {
    DeviceGuard g(device);
    XCK(cudaIpcCloseMemHandle(d_ptr));
    return XPIR_OK;
}

int xpir_device_sync(int device) {
    DeviceGuard g(device);
    XCK(cudaDeviceSynchronize());
    return XPIR_OK;
}

int xpir_store_create(int device, uint32_t N, uint32_t S, uint32_t lo, uint32_t hi,
                      xpir_store** out) {
    if (!out) return fail(XPIR_EINVAL, "store_create: null out");
    if (N == 0 || S == 0) return fail(XPIR_EINVAL, "store_create: empty geometry");
    if (lo >= hi || hi > N) return fail(XPIR_EINVAL, "store_create: bad shard range");
    if (lo % 8 != 0 || (hi % 8 != 0 && hi != N))
        return fail(XPIR_EINVAL, "store_create: shard bounds must be multiples of 8 buckets");
    int ndev = 0;
    XCK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(XPIR_EINVAL, "store_create: bad device");
    DeviceGuard g(device);
    auto* st = new xpir_store;
    st->device = device;
    st->N = N;
    st->S = S;
    st->lo = lo;
    st->hi = hi;
    cudaError_t e = cudaMalloc(&st->data, std::max<uint64_t>(st->bytes(), 16));
    if (e != cudaSuccess) {
        delete st;
        return fail(XPIR_ENOMEM, std::string("store_create: ") + cudaGetErrorString(e));
    }
    e = cudaStreamCreateWithFlags(&st->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        cudaFree(st->data);
        delete st;
        return fail(XPIR_ECUDA, cudaGetErrorString(e));
    }
    *out = st;
    return XPIR_OK;
}

int xpir_store_destroy(xpir_store* st) {
    if (!st) return XPIR_OK;
    DeviceGuard g(st->device);
    cudaStreamSynchronize(st->stream);
    cudaFree(st->data);
    st->q.release();
    st->out.release();
    st->seeds.release();
    st->masks.release();
    st->qwin.release();
    for (auto& e : st->qwin_by_stream) {
        e.second->release();
        delete e.second;
    }
    st->qx.release();
    st->idx.release();
    cudaStreamDestroy(st->stream);
    delete st;
    return XPIR_OK;
}

int xpir_store_upload(xpir_store* st, const uint8_t* host, uint64_t epoch) {
    if (!st || !host) return fail(XPIR_EINVAL, "store_upload: null argument");
    std::lock_guard<std::mutex> lk(st->mu);
    DeviceGuard g(st->device);
    XCK(cudaMemcpyAsync(st->data, host, st->bytes(), cudaMemcpyHostToDevice, st->stream));
    XCK(cudaStreamSynchronize(st->stream));
    st->epoch = epoch;
    return XPIR_OK;
}

int xpir_store_upload_dev(xpir_store* st, const void* src, uint64_t epoch, void* stream) {
    if (!st || !src) return fail(XPIR_EINVAL, "store_upload_dev: null argument");
    DeviceGuard g(st->device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : st->stream;
    XCK(cudaMemcpyAsync(st->data, src, st->bytes(), cudaMemcpyDeviceToDevice, s));
    st->epoch = epoch;
    return XPIR_OK;
}

int xpir_store_fill_keystream(xpir_store* st, const uint8_t key[32], uint64_t nonce,
                              uint64_t epoch, void* stream) {
    if (!st || !key) return fail(XPIR_EINVAL, "store_fill_keystream: null argument");
    DeviceGuard g(st->device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : st->stream;
    XCK(launch_keystream(key, nonce, uint64_t(st->lo) * st->S, st->data, st->bytes(), s));
    count_launches(1);
    if (!stream) XCK(cudaStreamSynchronize(s));
    st->epoch = epoch;
    return XPIR_OK;
}

int xpir_store_info(const xpir_store* st, uint32_t* N, uint32_t* S, uint32_t* lo, uint32_t* hi,
                    uint64_t* epoch, void** dev) {
    if (!st) return fail(XPIR_EINVAL, "store_info: null store");
    if (N) *N = st->N;
    if (S) *S = st->S;
    if (lo) *lo = st->lo;
    if (hi) *hi = st->hi;
    if (epoch) *epoch = st->epoch;
    if (dev) *dev = st->data;
    return XPIR_OK;
}

int xpir_store_download(const xpir_store* st, uint64_t offset, uint64_t len, uint8_t* host) {
    if (!st || (len && !host)) return fail(XPIR_EINVAL, "store_download: null argument");
    if (offset > st->bytes() || len > st->bytes() - offset)
        return fail(XPIR_EINVAL, "store_download: range outside the shard");
    DeviceGuard g(st->device);
    XCK(cudaStreamSynchronize(st->stream));
    if (len) XCK(cudaMemcpy(host, st->data + offset, len, cudaMemcpyDeviceToHost));
    return XPIR_OK;
}

uint64_t xpir_query_window_bytes(const xpir_store* st) {
    return st ? round16(st->nbytes_window()) + 16 : 0;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Scan dispatch. Kernel choice: 2 = M4RM (S % 128 == 0, B >= 128; group-major
// queries), 1 = direct select-XOR (S % 16 == 0; row-major query window),
// 3 = byte-granular (any S).
// ---------------------------------------------------------------------------
// Batch-size crossovers from the config-5 sweep: the byte-table
// M4RM kernels from 128 requests; below, the direct kernel. The warp-private
// nibble-table kernel (6) measured slower than direct at every B in [8, 128)
// (latency-bound), so it is selectable but not chosen automatically.
static uint32_t g_nib_min_batch = 0xffffffffu;
static uint32_t g_k4_min_batch = 24;   // nibble-table M4RM (kernel 7) from here
static uint32_t g_m4_min_batch = 257;  // byte-table M4RM (kernels 2/5) from here
static uint32_t g_q_min_batch = 2048;  // quad-table full-TMEM M4RM (kernel 8) from here

static int choose_kernel(const xpir_store* st, uint32_t B) {
    int k;
    {
        std::lock_guard<std::mutex> lk(g_opts_mu);
        k = g_opts.kernel;
    }
    if (st->S % 16 != 0) return 3;
    const bool m4_ok = (st->S % 128) == 0;
    const bool q_ok = (st->S % 32) == 0;
    if (k == 4 || k == 5) k = 2;  // forced M4RM variants (registers-only / TMEM accumulators)
    if (k == 0) {
        // B >= 2048: quad tables (8) or the half-TMEM 128-byte-column kernel (2 -> 5),
        // whichever the sweep-calibrated cost model says is faster for this B
        if (q_ok && B >= g_q_min_batch) {
            const double c5 = m4_ok ? double((uint64_t(B) + 2047) / 2048 * 2048) / 3.0 : 1e300;
            return m4rm_q_cost(B, nullptr) < c5 ? 8 : 2;
        }
        k = !m4_ok ? 1 : B >= g_m4_min_batch ? 2 : B >= g_k4_min_batch ? 7 : B >= g_nib_min_batch ? 6 : 1;
    }
    if ((k == 2 || k == 6 || k == 7) && !m4_ok) k = 1;
    if (k == 8 && !q_ok) k = 1;
    return k;
}

static int run_m4(xpir_store* st, const uint8_t* qT, uint64_t qstride, uint32_t B, uint8_t* d_out,
                  cudaStream_t s, int kernel) {
    int cps, variant;
    {
        std::lock_guard<std::mutex> lk(g_opts_mu);
        cps = g_opts.ctas_per_sm;
        variant = g_opts.kernel == 4 ? 1 : g_opts.kernel == 5 ? 2 : 0;
    }
    M4Args a{st->data, st->nb(), st->S, qT, qstride, B, d_out, s};
    cudaEvent_t ev;
    if (kernel == 8) {  // quad-interleaved 32-byte-column tables, full-TMEM accumulators
        timing_begin(s, &ev);
        XCK(launch_scan_m4rm_q(a, num_sms(st->device)));
        timing_end(s, ev);
        count_launches(1);
        g_last_kernel = 8;
        return XPIR_OK;
    }
    if (kernel == 7) {  // nibble tables
        timing_begin(s, &ev);
        XCK(launch_scan_m4rm4(a, num_sms(st->device)));
        timing_end(s, ev);
        count_launches(1);
        g_last_kernel = 7;
        return XPIR_OK;
    }
    timing_begin(s, &ev);
    XCK(launch_scan_m4rm(a, cps, num_sms(st->device), variant));
    timing_end(s, ev);
    count_launches(1);
    // 2 = M4RM with register accumulators, 5 = M4RM with half-TMEM accumulators
    g_last_kernel = (variant == 2 || (variant == 0 && B >= 2048)) ? 5 : 2;
    return XPIR_OK;
}

// qwin: row-major query rows already offset to the shard's first byte.
static int run_rows(xpir_store* st, int kernel, const uint8_t* qwin, uint64_t stride, uint32_t B,
                    uint8_t* d_out, cudaStream_t s) {
    ScanArgs a{st->data, st->nb(), st->S, qwin, stride, B, d_out, s};
    if (kernel == 3) {
        XCK(launch_scan_bytes(a));
        count_launches(1);
        g_last_kernel = 3;
        return XPIR_OK;
    }
    if (kernel == 6) {
        cudaEvent_t ev;
        timing_begin(s, &ev);
        XCK(launch_scan_nib(a, num_sms(st->device)));
        timing_end(s, ev);
        count_launches(1);
        g_last_kernel = 6;
        return XPIR_OK;
    }
    // direct: CTAs XOR their partials straight into `out` (no partial buffer)
    uint32_t nsplit = 0;
    cudaEvent_t ev;
    timing_begin(s, &ev);
    XCK(launch_scan_direct(a, num_sms(st->device), &nsplit));
    timing_end(s, ev);
    count_launches(1);
    g_last_kernel = 1;
    return XPIR_OK;
}

// Row-major query rows (device; `rows` points at row 0 byte 0 of the FULL vector).
static int scan_rows(xpir_store* st, const uint8_t* rows, uint64_t stride, uint32_t B,
                     const uint8_t* d_mask, uint8_t* d_out, cudaStream_t s) {
    XCK(launch_init_out(d_out, B, st->S, d_mask, false, s));
    count_launches(1);
    if (B == 0) return XPIR_OK;
    const int k = choose_kernel(st, B);
    const uint64_t blo = st->byte_lo(), nbw = st->nbytes_window();
    if (k != 2 && k != 7 && k != 8) return run_rows(st, k, rows + blo, stride, B, d_out, s);
    const uint64_t qs = m4rm_qstride(B);
    DevBuf& qw = st->qwin_for(s);
    XCK(qw.ensure(m4rm_qrows(nbw) * qs));
    XCK(launch_transpose_q(rows, stride, blo, nbw, B, qw.as<uint8_t>(), qs, s, k == 8));
    count_launches(1);
    return run_m4(st, qw.as<uint8_t>(), qs, B, d_out, s, k);
}

extern "C" {

int xpir_answer_batch_dev(xpir_store* st, const uint8_t* d_q, uint64_t q_stride, uint32_t q_bits,
                          uint32_t B, const uint8_t* d_mask, uint8_t* d_out, void* stream) {
    if (!st) return fail(XPIR_EINVAL, "answer_batch: null store");
    if (q_bits != st->N) return fail(XPIR_EINVAL, "answer_batch: query length mismatch");
    if (B && (!d_q || !d_out)) return fail(XPIR_EINVAL, "answer_batch: null buffer");
    if (B && q_stride < (uint64_t(st->N) + 7) / 8)
        return fail(XPIR_EINVAL, "answer_batch: query stride shorter than the vector");
    DeviceGuard g(st->device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : st->stream;
    return scan_rows(st, d_q, q_stride, B, d_mask, d_out, s);
}

int xpir_answer_batch_seeded_dev(xpir_store* st, const uint8_t* d_seeds, uint32_t B,
                                 const uint8_t* d_mask, uint8_t* d_out, void* stream) {
    if (!st) return fail(XPIR_EINVAL, "answer_batch_seeded: null store");
    if (B && (!d_seeds || !d_out)) return fail(XPIR_EINVAL, "answer_batch_seeded: null buffer");
    DeviceGuard g(st->device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : st->stream;
    XCK(launch_init_out(d_out, B, st->S, d_mask, false, s));
    count_launches(1);
    if (B == 0) return XPIR_OK;
    const int k = choose_kernel(st, B);
    const uint64_t blo = st->byte_lo(), nbw = st->nbytes_window();
    // K2: expand only this shard's window of every request's selection vector,
    // straight into the layout the chosen scan kernel reads.
    if (k == 2 || k == 7 || k == 8) {
        const uint64_t qs = m4rm_qstride(B);
        DevBuf& qw = st->qwin_for(s);
        XCK(qw.ensure(m4rm_qrows(nbw) * qs));
        XCK(launch_expand_T(d_seeds, B, blo, nbw, qw.as<uint8_t>(), qs, s, k == 8));
        count_launches(1);
        return run_m4(st, qw.as<uint8_t>(), qs, B, d_out, s, k);
    }
    const uint64_t ws = xpir_query_window_bytes(st);
    DevBuf& qw = st->qwin_for(s);
    XCK(qw.ensure(ws * B));
    XCK(launch_expand(d_seeds, B, blo, nbw, qw.as<uint8_t>(), ws, s));
    count_launches(1);
    return run_rows(st, k, qw.as<uint8_t>(), ws, B, d_out, s);
}

int xpir_answer_batch(xpir_store* st, const uint8_t* q, uint64_t q_stride, uint32_t q_bits,
                      uint32_t B, const uint8_t* mask_seeds, uint8_t* out) {
    if (!st) return fail(XPIR_EINVAL, "answer_batch: null store");
    if (q_bits != st->N) return fail(XPIR_EINVAL, "answer_batch: query length mismatch");
    if (B == 0) return XPIR_OK;
    if (!q || !out) return fail(XPIR_EINVAL, "answer_batch: null buffer");
    if (q_stride < (uint64_t(st->N) + 7) / 8)
        return fail(XPIR_EINVAL, "answer_batch: query stride shorter than the vector");
    std::lock_guard<std::mutex> lk(st->mu);
    DeviceGuard g(st->device);
    cudaStream_t s = st->stream;
    const uint64_t blo = st->byte_lo(), nbw = st->nbytes_window();
    const uint64_t ws = round16(nbw) + 16;
    XCK(st->q.ensure(ws * B));
    // H2D of the shard's window of every row (pitched copy); rows start at byte 0
    XCK(cudaMemcpy2DAsync(st->q.p, ws, q + blo, q_stride, nbw, B, cudaMemcpyHostToDevice, s));
    const uint8_t* dm = nullptr;
    if (mask_seeds) {
        XCK(st->masks.ensure(uint64_t(B) * 32));
        XCK(cudaMemcpyAsync(st->masks.p, mask_seeds, uint64_t(B) * 32, cudaMemcpyHostToDevice, s));
        dm = st->masks.as<uint8_t>();
    }
    const uint64_t ob = uint64_t(B) * st->S;
    XCK(st->out.ensure(ob));
    uint8_t* dout = st->out.as<uint8_t>();
    XCK(launch_init_out(dout, B, st->S, dm, false, s));
    count_launches(1);
    const int k = choose_kernel(st, B);
    int rc;
    if (k == 2 || k == 7 || k == 8) {
        const uint64_t qs = m4rm_qstride(B);
        XCK(st->qwin.ensure(m4rm_qrows(nbw) * qs));
        XCK(launch_transpose_q(st->q.as<uint8_t>(), ws, 0, nbw, B, st->qwin.as<uint8_t>(), qs, s, k == 8));
        count_launches(1);
        rc = run_m4(st, st->qwin.as<uint8_t>(), qs, B, dout, s, k);
    } else {
        rc = run_rows(st, k, st->q.as<uint8_t>(), ws, B, dout, s);
    }
    if (rc) return rc;
    XCK(cudaMemcpyAsync(out, st->out.p, ob, cudaMemcpyDeviceToHost, s));
    XCK(cudaStreamSynchronize(s));
    return XPIR_OK;
}

// Seed-compressed read shares: a batch where request r is
// either an explicit selection vector or a 32-byte PRG seed whose prng_expand is
// the vector (crypto.cpp:35-45). Explicit rows and seeds arrive compacted, in
// request order; only they cross PCIe. Both are placed into one row-major
// window buffer on device (row scatter + row-mapped K2), then scanned as one batch.
int xpir_answer_batch_mixed(xpir_store* st, uint32_t B, const uint8_t* is_seed, const uint8_t* seeds,
                            const uint8_t* q, uint64_t q_stride, uint32_t q_bits, const uint8_t* mask_seeds,
                            uint8_t* out) {
    if (!st) return fail(XPIR_EINVAL, "answer_batch_mixed: null store");
    if (q_bits != st->N) return fail(XPIR_EINVAL, "answer_batch_mixed: query length mismatch");
    if (B == 0) return XPIR_OK;
    if (!is_seed || !out) return fail(XPIR_EINVAL, "answer_batch_mixed: null buffer");
    std::vector<uint32_t> idx(B);
    uint32_t ns = 0, ne = 0;
    for (uint32_t r = 0; r < B; ++r) (is_seed[r] ? ns : ne) += 1;
    for (uint32_t r = 0, a = 0, b = 0; r < B; ++r) idx[is_seed[r] ? ne + a++ : b++] = r;  // [explicit | seeded]
    if (ns && !seeds) return fail(XPIR_EINVAL, "answer_batch_mixed: seeded requests without seeds");
    if (ne && (!q || q_stride < (uint64_t(st->N) + 7) / 8))
        return fail(XPIR_EINVAL, "answer_batch_mixed: explicit rows missing or stride too short");
    std::lock_guard<std::mutex> lk(st->mu);
    DeviceGuard g(st->device);
    cudaStream_t s = st->stream;
    const uint64_t blo = st->byte_lo(), nbw = st->nbytes_window();
    const uint64_t ws = round16(nbw) + 16;
    XCK(st->q.ensure(ws * B));
    XCK(st->idx.ensure(4 * uint64_t(B)));
    XCK(cudaMemcpyAsync(st->idx.p, idx.data(), 4 * uint64_t(B), cudaMemcpyHostToDevice, s));
    const uint32_t* d_idx = st->idx.as<uint32_t>();
    if (ne) {  // explicit rows: H2D of the shard window of each, then into their request rows
        XCK(st->qx.ensure(ws * ne));
        XCK(cudaMemcpy2DAsync(st->qx.p, ws, q + blo, q_stride, nbw, ne, cudaMemcpyHostToDevice, s));
        XCK(launch_scatter_rows(st->qx.as<uint8_t>(), ws, ne, d_idx, st->q.as<uint8_t>(), ws, nbw, s));
        count_launches(1);
    }
    if (ns) {  // seeded rows: K2 straight into their request rows (this shard's window only)
        XCK(st->seeds.ensure(uint64_t(ns) * 32));
        XCK(cudaMemcpyAsync(st->seeds.p, seeds, uint64_t(ns) * 32, cudaMemcpyHostToDevice, s));
        XCK(launch_expand(st->seeds.as<uint8_t>(), ns, blo, nbw, st->q.as<uint8_t>(), ws, s, d_idx + ne));
        count_launches(1);
    }
    const uint8_t* dm = nullptr;
    if (mask_seeds) {
        XCK(st->masks.ensure(uint64_t(B) * 32));
        XCK(cudaMemcpyAsync(st->masks.p, mask_seeds, uint64_t(B) * 32, cudaMemcpyHostToDevice, s));
        dm = st->masks.as<uint8_t>();
    }
    const uint64_t ob = uint64_t(B) * st->S;
    XCK(st->out.ensure(ob));
    uint8_t* dout = st->out.as<uint8_t>();
    XCK(launch_init_out(dout, B, st->S, dm, false, s));
    count_launches(1);
    const int k = choose_kernel(st, B);
    int rc;
    if (k == 2 || k == 7 || k == 8) {
        const uint64_t qs = m4rm_qstride(B);
        XCK(st->qwin.ensure(m4rm_qrows(nbw) * qs));
        XCK(launch_transpose_q(st->q.as<uint8_t>(), ws, 0, nbw, B, st->qwin.as<uint8_t>(), qs, s, k == 8));
        count_launches(1);
        rc = run_m4(st, st->qwin.as<uint8_t>(), qs, B, dout, s, k);
    } else {
        rc = run_rows(st, k, st->q.as<uint8_t>(), ws, B, dout, s);
    }
    if (rc) return rc;
    XCK(cudaMemcpyAsync(out, st->out.p, ob, cudaMemcpyDeviceToHost, s));
    XCK(cudaStreamSynchronize(s));
    return XPIR_OK;
}

int xpir_answer_batch_seeded(xpir_store* st, const uint8_t* seeds, uint32_t B,
                             const uint8_t* mask_seeds, uint8_t* out) {
    if (!st) return fail(XPIR_EINVAL, "answer_batch_seeded: null store");
    if (B == 0) return XPIR_OK;
    if (!seeds || !out) return fail(XPIR_EINVAL, "answer_batch_seeded: null buffer");
    std::lock_guard<std::mutex> lk(st->mu);
    DeviceGuard g(st->device);
    cudaStream_t s = st->stream;
    XCK(st->seeds.ensure(uint64_t(B) * 32));
    XCK(cudaMemcpyAsync(st->seeds.p, seeds, uint64_t(B) * 32, cudaMemcpyHostToDevice, s));
    const uint8_t* dm = nullptr;
    if (mask_seeds) {
        XCK(st->masks.ensure(uint64_t(B) * 32));
        XCK(cudaMemcpyAsync(st->masks.p, mask_seeds, uint64_t(B) * 32, cudaMemcpyHostToDevice, s));
        dm = st->masks.as<uint8_t>();
    }
    const uint64_t ob = uint64_t(B) * st->S;
    XCK(st->out.ensure(ob));
    int rc = xpir_answer_batch_seeded_dev(st, st->seeds.as<uint8_t>(), B, dm, st->out.as<uint8_t>(), s);
    if (rc) return rc;
    XCK(cudaMemcpyAsync(out, st->out.p, ob, cudaMemcpyDeviceToHost, s));
    XCK(cudaStreamSynchronize(s));
    return XPIR_OK;
}

int xpir_answer_batch_seeded_peer_dev(xpir_store* st, const uint8_t* d_seeds, uint32_t B,
                                      uint8_t* const* out_ptrs, const uint32_t* row_bounds, uint32_t n_ranks,
                                      void* stream) {
    if (!st) return fail(XPIR_EINVAL, "answer_batch_seeded_peer: null store");
    if (n_ranks < 1 || n_ranks > 8) return fail(XPIR_EINVAL, "answer_batch_seeded_peer: 1..8 ranks");
    if (!out_ptrs || !row_bounds || (B && !d_seeds)) return fail(XPIR_EINVAL, "answer_batch_seeded_peer: null");
    if (row_bounds[0] != 0 || row_bounds[n_ranks] != B)
        return fail(XPIR_EINVAL, "answer_batch_seeded_peer: row bounds must cover [0, B)");
    if (st->S % 32 != 0 || B < 2048)
        return fail(XPIR_EINVAL, "answer_batch_seeded_peer: fused reduce needs S % 32 == 0 and B >= 2048");
    DeviceGuard g(st->device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : st->stream;
    const uint64_t blo = st->byte_lo(), nbw = st->nbytes_window();
    const uint64_t qs = m4rm_qstride(B);
    DevBuf& qw = st->qwin_for(s);
    XCK(qw.ensure(m4rm_qrows(nbw) * qs));
    XCK(launch_expand_T(d_seeds, B, blo, nbw, qw.as<uint8_t>(), qs, s, true));  // the fused path always runs kernel 8
    M4Args a{st->data, st->nb(), st->S, qw.as<uint8_t>(), qs, B, out_ptrs[0], s};
    a.peers.n = n_ranks;
    for (uint32_t k = 0; k < n_ranks; ++k) {
        a.peers.ptr[k] = out_ptrs[k];
        a.peers.bound[k] = row_bounds[k];
    }
    a.peers.bound[n_ranks] = row_bounds[n_ranks];
    cudaEvent_t ev;
    timing_begin(s, &ev);
    XCK(launch_scan_m4rm_q(a, num_sms(st->device)));
    timing_end(s, ev);
    count_launches(2);
    g_last_kernel = 8;
    return XPIR_OK;
}

int xpir_init_rows_dev(int device, uint8_t* d_out, uint32_t r0, uint32_t r1, uint32_t S,
                       const uint8_t* d_mask_seeds, void* stream) {
    if (r1 < r0 || (r1 > r0 && !d_out)) return fail(XPIR_EINVAL, "init_rows: bad range");
    DeviceGuard g(device);
    XCK(launch_init_out(d_out + uint64_t(r0) * S, r1 - r0, S, d_mask_seeds ? d_mask_seeds + uint64_t(r0) * 32 : nullptr,
                        false, static_cast<cudaStream_t>(stream)));
    count_launches(1);
    return XPIR_OK;
}

int xpir_expand_queries_dev(int device, const uint8_t* d_seeds, uint32_t B, uint64_t byte_lo,
                            uint64_t nbytes, uint8_t* d_q, uint64_t q_stride, void* stream) {
    if (B && (!d_seeds || !d_q)) return fail(XPIR_EINVAL, "expand_queries: null buffer");
    if (q_stride < nbytes) return fail(XPIR_EINVAL, "expand_queries: stride < nbytes");
    DeviceGuard g(device);
    XCK(launch_expand(d_seeds, B, byte_lo, nbytes, d_q, q_stride, static_cast<cudaStream_t>(stream)));
    count_launches(1);
    return XPIR_OK;
}

int xpir_mask_answer(const uint8_t* ans, uint64_t len, const uint8_t seed[32], uint8_t* out) {
    if (!seed || (len && (!ans || !out))) return fail(XPIR_EINVAL, "mask_answer: null buffer");
    if (!len) return XPIR_OK;
    if (len > 0xffffffffull) return fail(XPIR_EINVAL, "mask_answer: answer too long");
    uint8_t* d = nullptr;
    XCK(cudaMalloc(&d, len + 32));
    cudaError_t e = cudaMemcpy(d, ans, len, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d + len, seed, 32, cudaMemcpyHostToDevice);
    // one "request" of S = len bytes: out = ans ^ pad
    if (e == cudaSuccess) e = launch_init_out(d, 1, uint32_t(len), d + len, true, nullptr);
    count_launches(1);
    if (e == cudaSuccess) e = cudaMemcpy(out, d, len, cudaMemcpyDeviceToHost);
    cudaFree(d);
    XCK(e);
    return XPIR_OK;
}

int xpir_mask_dev(int device, uint8_t* d_out, const uint8_t* d_mask, uint32_t B, uint32_t S,
                  void* stream) {
    if (B && (!d_out || !d_mask)) return fail(XPIR_EINVAL, "mask: null buffer");
    DeviceGuard g(device);
    XCK(launch_init_out(d_out, B, S, d_mask, true, static_cast<cudaStream_t>(stream)));
    count_launches(1);
    return XPIR_OK;
}

int xpir_xor_reduce_dev(int device, uint8_t* d_dst, const uint8_t* const* d_srcs, uint32_t nsrc,
                        uint64_t bytes, void* stream) {
    if (nsrc && (!d_dst || !d_srcs)) return fail(XPIR_EINVAL, "xor_reduce: null buffer");
    DeviceGuard g(device);
    XCK(launch_xor_reduce(d_dst, d_srcs, nsrc, bytes, num_sms(device), static_cast<cudaStream_t>(stream)));
    count_launches(1);
    return XPIR_OK;
}

// ---------------------------------------------------------------------------
// primitives
// ---------------------------------------------------------------------------
int xpir_prng_expand(const uint8_t seed[32], uint8_t* out, uint64_t len) {
    if (!seed || (len && !out)) return fail(XPIR_EINVAL, "prng_expand: null buffer");
    if (!len) return XPIR_OK;
    uint8_t* d = nullptr;
    XCK(cudaMalloc(&d, len));
    cudaError_t e = launch_keystream(seed, 0, 0, d, len, nullptr);
    count_launches(1);
    if (e == cudaSuccess) e = cudaMemcpy(out, d, len, cudaMemcpyDeviceToHost);
    cudaFree(d);
    XCK(e);
    return XPIR_OK;
}

int xpir_keystream_dev(int device, const uint8_t key[32], uint64_t nonce, uint64_t byte_offset,
                       uint8_t* d_out, uint64_t len, void* stream) {
    if (!key || (len && !d_out)) return fail(XPIR_EINVAL, "keystream: null buffer");
    DeviceGuard g(device);
    XCK(launch_keystream(key, nonce, byte_offset, d_out, len, static_cast<cudaStream_t>(stream)));
    count_launches(1);
    return XPIR_OK;
}

int xpir_keystream_rows_dev(int device, const uint8_t key[32], uint64_t nonce0, uint32_t rows,
                            uint64_t len, uint8_t* d_out, uint64_t row_stride, void* stream) {
    if (!key || (rows && len && !d_out)) return fail(XPIR_EINVAL, "keystream_rows: null buffer");
    if (row_stride < len) return fail(XPIR_EINVAL, "keystream_rows: stride < len");
    DeviceGuard g(device);
    XCK(launch_keystream_rows(key, nonce0, rows, len, d_out, row_stride, static_cast<cudaStream_t>(stream)));
    count_launches(1);
    return XPIR_OK;
}

int xpir_prf_batch(const uint8_t key[16], const uint64_t* inputs, uint64_t n, uint64_t modulus,
                   uint64_t* out) {
    if (modulus == 0) return fail(XPIR_EINVAL, "prf: modulus must be positive");
    if (!key || (n && (!inputs || !out))) return fail(XPIR_EINVAL, "prf: null buffer");
    if (!n) return XPIR_OK;
    uint64_t* d = nullptr;
    XCK(cudaMalloc(&d, 16 * n));
    cudaError_t e = cudaMemcpy(d, inputs, 8 * n, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = launch_prf(ld64le(key), ld64le(key + 8), d, n, modulus, d + n, nullptr, nullptr);
    count_launches(1);
    if (e == cudaSuccess) e = cudaMemcpy(out, d + n, 8 * n, cudaMemcpyDeviceToHost);
    cudaFree(d);
    XCK(e);
    return XPIR_OK;
}

int xpir_prf_batch_dev(int device, const uint8_t key[16], const uint64_t* d_in, uint64_t n, uint64_t modulus,
                       uint64_t* d_out, uint32_t* d_out32, void* stream) {
    if (modulus == 0) return fail(XPIR_EINVAL, "prf: modulus must be positive");
    if (!key || (n && !d_in)) return fail(XPIR_EINVAL, "prf: null buffer");
    DeviceGuard g(device);
    XCK(launch_prf(ld64le(key), ld64le(key + 8), d_in, n, modulus, d_out, d_out32,
                   static_cast<cudaStream_t>(stream)));
    count_launches(1);
    return XPIR_OK;
}

int xpir_make_interest_batch(uint32_t m_bits, uint32_t h, const uint8_t id[16],
                             const uint64_t* seqs, uint64_t n, uint32_t* out) {
    if (m_bits == 0) return fail(XPIR_EINVAL, "bloom_positions: m_bits must be positive");
    if (!id || (n && (!seqs || !out))) return fail(XPIR_EINVAL, "make_interest: null buffer");
    if (!n || !h) return XPIR_OK;
    uint64_t* ds = nullptr;
    uint32_t* dp = nullptr;
    XCK(cudaMalloc(&ds, 8 * n));
    cudaError_t e = cudaMalloc(&dp, 4 * n * h);
    if (e == cudaSuccess) e = cudaMemcpy(ds, seqs, 8 * n, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = launch_interest(id, ds, n, h, m_bits, dp, nullptr, nullptr);
    count_launches(1);
    if (e == cudaSuccess) e = cudaMemcpy(out, dp, 4 * n * h, cudaMemcpyDeviceToHost);
    cudaFree(ds);
    cudaFree(dp);
    XCK(e);
    return XPIR_OK;
}

int xpir_bloom_positions(const uint8_t* item, uint64_t len, uint32_t h, uint32_t m_bits,
                         uint32_t* out) {
    if (m_bits == 0) return fail(XPIR_EINVAL, "bloom_positions: m_bits must be positive");
    if (len > 120) return fail(XPIR_EINVAL, "bloom_positions: device port takes items <= 120 bytes");
    if ((len && !item) || (h && !out)) return fail(XPIR_EINVAL, "bloom_positions: null buffer");
    if (!h) return XPIR_OK;
    uint8_t* d = nullptr;
    XCK(cudaMalloc(&d, 128 + 4 * uint64_t(h)));
    cudaError_t e = len ? cudaMemcpy(d, item, len, cudaMemcpyHostToDevice) : cudaSuccess;
    uint32_t* dp = reinterpret_cast<uint32_t*>(d + 128);
    if (e == cudaSuccess) e = launch_bloom_item(d, uint32_t(len), h, m_bits, dp, nullptr);
    count_launches(1);
    if (e == cudaSuccess) e = cudaMemcpy(out, dp, 4 * uint64_t(h), cudaMemcpyDeviceToHost);
    cudaFree(d);
    XCK(e);
    return XPIR_OK;
}

int xpir_blake2b(const uint8_t* data, uint64_t len, uint32_t outlen, uint8_t* out) {
    if (outlen < 1 || outlen > 64) return fail(XPIR_EINVAL, "blake2b: outlen must be 1..64");
    if ((len && !data) || !out) return fail(XPIR_EINVAL, "blake2b: null buffer");
    HostBlake2b h(outlen);
    h.update(data, len);
    h.final(out);
    return XPIR_OK;
}

}  // extern "C"

// ===========================================================================
// cuckoo table
// ===========================================================================
struct xpir_table {
    int device;
    uint8_t seed[32];
    CuckooDev d{};
    CuckooState h{};
    CuckooState* dstate = nullptr;
    uint8_t* data = nullptr;  // payloads of buckets [lo, hi)
    uint32_t lo = 0, hi = 0;  // a payload shard of the logical table (metadata is whole)
    cudaStream_t stream = nullptr;
    DevBuf in_b1, in_b2, in_payload, in_reports, gather;
    CuckooParScratch par;
    bool parallel_prefix = true;  // XPIR_CUCKOO_SEQUENTIAL=1 disables (A/B checks)
    std::mutex mu;
    uint64_t slots() const { return uint64_t(d.buckets) * d.depth; }
    uint64_t data_bytes() const { return uint64_t(hi - lo) * d.depth * d.item; }
    bool sharded() const { return lo != 0 || hi != d.buckets; }
};

static const uint32_t DRAW_CAP = 1u << 16;

static void table_free_all(xpir_table* t) {
    cudaFree(t->d.used);
    cudaFree(t->d.beta1);
    cudaFree(t->d.beta2);
    cudaFree(t->d.stamp);
    cudaFree(t->d.origin);
    cudaFree(t->d.touched_mark);
    cudaFree(t->d.touched);
    cudaFree(t->d.mod_batch);
    cudaFree(t->d.chain_pre);
    cudaFree(t->d.fifo);
    cudaFree(t->d.draws);
    cudaFree(t->dstate);
    cudaFree(t->data);
    t->in_b1.release();
    t->in_b2.release();
    t->in_payload.release();
    t->in_reports.release();
    t->gather.release();
    t->par.release();
    if (t->stream) cudaStreamDestroy(t->stream);
}

extern "C" {

int xpir_table_create(int device, uint32_t buckets, uint32_t depth, uint64_t capacity,
                      uint64_t item_size, const uint8_t seed[32], xpir_table** out) {
    return xpir_table_create_shard(device, buckets, depth, capacity, item_size, seed, 0, buckets, out);
}

int xpir_table_create_shard(int device, uint32_t buckets, uint32_t depth, uint64_t capacity, uint64_t item_size,
                            const uint8_t seed[32], uint32_t lo, uint32_t hi, xpir_table** out) {
    if (!out || !seed) return fail(XPIR_EINVAL, "table_create: null argument");
    if (buckets == 0 || depth == 0 || item_size == 0)  // cuckoo.cpp:15-16
        return fail(XPIR_EINVAL, "cuckoo: table dimensions must be positive");
    if (capacity == 0 || capacity > uint64_t(buckets) * depth)  // cuckoo.cpp:17-18
        return fail(XPIR_EINVAL, "cuckoo: capacity must be in [1, buckets*depth]");
    if (uint64_t(buckets) * depth >= (uint64_t(1) << 32))
        return fail(XPIR_EINVAL, "cuckoo: more than 2^32 slots");
    if (lo >= hi || hi > buckets) return fail(XPIR_EINVAL, "table_create: bad shard bucket range");
    int ndev = 0;
    XCK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(XPIR_EINVAL, "table_create: bad device");
    DeviceGuard g(device);
    auto* t = new xpir_table;
    t->device = device;
    std::memcpy(t->seed, seed, 32);
    t->d.buckets = buckets;
    t->d.depth = depth;
    t->d.capacity = capacity;
    t->d.item = item_size;
    const uint64_t slots = t->slots();
    uint64_t fc = 1;
    while (fc < 2 * slots + 1024) fc <<= 1;
    t->d.fifo_cap = fc;
    t->d.draw_cap = DRAW_CAP;
    cudaError_t e = cudaSuccess;
    auto M = [&](void** p, size_t n) {
        if (e == cudaSuccess) e = cudaMalloc(p, std::max<size_t>(n, 16));
        if (e == cudaSuccess) e = cudaMemset(*p, 0, std::max<size_t>(n, 16));
    };
    M(reinterpret_cast<void**>(&t->d.used), slots);
    M(reinterpret_cast<void**>(&t->d.beta1), 4 * slots);
    M(reinterpret_cast<void**>(&t->d.beta2), 4 * slots);
    M(reinterpret_cast<void**>(&t->d.stamp), 8 * slots);
    M(reinterpret_cast<void**>(&t->d.origin), 8 * slots);
    M(reinterpret_cast<void**>(&t->d.touched_mark), 4 * slots);
    M(reinterpret_cast<void**>(&t->d.touched), 4 * slots);
    M(reinterpret_cast<void**>(&t->d.mod_batch), 4 * slots);
    M(reinterpret_cast<void**>(&t->d.chain_pre), 8 * 3 * 512);
    M(reinterpret_cast<void**>(&t->d.fifo), 8 * fc);
    M(reinterpret_cast<void**>(&t->d.draws), 8 * uint64_t(DRAW_CAP));
    M(reinterpret_cast<void**>(&t->dstate), sizeof(CuckooState));
    t->lo = lo;
    t->hi = hi;
    M(reinterpret_cast<void**>(&t->data), uint64_t(hi - lo) * depth * item_size);
    if (e == cudaSuccess) e = cudaMemset(t->d.fifo, 0xff, 8 * fc);  // -1: no entry
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        table_free_all(t);
        delete t;
        return fail(e == cudaErrorMemoryAllocation ? XPIR_ENOMEM : XPIR_ECUDA,
                    std::string("table_create: ") + cudaGetErrorString(e));
    }
    t->h = CuckooState{};
    if (const char* ev = std::getenv("XPIR_CUCKOO_SEQUENTIAL")) t->parallel_prefix = ev[0] != '1';
    *out = t;
    return XPIR_OK;
}

int xpir_table_destroy(xpir_table* t) {
    if (!t) return XPIR_OK;
    DeviceGuard g(t->device);
    cudaStreamSynchronize(t->stream);
    table_free_all(t);
    delete t;
    return XPIR_OK;
}

int xpir_table_insert_batch_dev(xpir_table* t, const uint32_t* d_b1, const uint32_t* d_b2,
                                const uint8_t* d_payload, uint64_t n, uint32_t* d_reports,
                                void* stream) {
    if (!t) return fail(XPIR_EINVAL, "table_insert: null table");
    if (n == 0) return XPIR_OK;
    if (!d_b1 || !d_b2 || !d_payload) return fail(XPIR_EINVAL, "table_insert: null buffer");
    if (t->sharded())
        return fail(XPIR_EINVAL, "table_insert: payload shard: use insert_walk + apply_gather (all shards) + apply_scatter");
    int rc = xpir_table_insert_walk_dev(t, d_b1, d_b2, n, d_reports, stream);
    if (rc) return rc;
    rc = xpir_table_apply_gather_dev(t, nullptr, stream);
    if (rc) return rc;
    return xpir_table_apply_scatter_dev(t, d_payload, stream);
}

int xpir_table_insert_walk_dev(xpir_table* t, const uint32_t* d_b1, const uint32_t* d_b2, uint64_t n,
                               uint32_t* d_reports, void* stream) {
    if (!t) return fail(XPIR_EINVAL, "table_insert: null table");
    DeviceGuard g(t->device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : t->stream;
    t->h.batch_id += 1;
    t->h.n_touched = 0;
    uint64_t i = 0;
    // K6a: the eviction-free, GC-free prefix of the round is placed in parallel
    // (exactly what the sequential walk would do); the walk continues from the
    // first insert that needs an eviction or a FIFO GC.
    if (t->parallel_prefix && n >= 64 && t->h.live < t->d.capacity) {
        const uint64_t room = t->d.capacity - t->h.live;
        uint64_t applied = 0;
        XCK(cuckoo_parallel_prefix(t->d, t->h, d_b1, d_b2, n < room ? n : room, d_reports, t->par, &applied, s));
        i = applied;
    }
    for (int guard = 0; i < n; ++guard) {
        if (t->h.rng_block + 1024 > t->h.draw_base + t->h.draw_count || guard == 0) {
            // (re)fill the draw window starting at the next unconsumed nonce
            t->h.draw_base = t->h.rng_block;
            t->h.draw_count = DRAW_CAP;
            XCK(launch_draws(t->seed, t->h.draw_base, DRAW_CAP, t->d.draws, s));
            count_launches(1);
        }
        XCK(cudaMemcpyAsync(t->dstate, &t->h, sizeof(CuckooState), cudaMemcpyHostToDevice, s));
        XCK(launch_cuckoo_walk(t->d, t->dstate, d_b1, d_b2, i, n, d_reports, s));
        count_launches(1);
        XCK(cudaMemcpyAsync(&t->h, t->dstate, sizeof(CuckooState), cudaMemcpyDeviceToHost, s));
        XCK(cudaStreamSynchronize(s));
        if (t->h.status == 2) return fail(XPIR_ESTATE, "table_insert: FIFO ring overflow");
        if (t->h.resume_at <= i && t->h.status != 1)
            return fail(XPIR_ESTATE, "table_insert: walk made no progress");
        i = t->h.resume_at;
        if (t->h.status == 1) t->h.draw_count = 0;  // force a refill
    }
    if (!stream) XCK(cudaStreamSynchronize(s));
    return XPIR_OK;
}

int xpir_table_apply_gather_dev(xpir_table* t, const xpir_shard_map* map, void* stream) {
    if (!t) return fail(XPIR_EINVAL, "table_apply: null table");
    ShardMap m{};
    if (map) {
        if (map->n > 8) return fail(XPIR_EINVAL, "table_apply: at most 8 shards");
        m.n = map->n;
        for (uint32_t k = 0; k <= map->n; ++k) m.lo[k] = map->bucket_lo[k];
        for (uint32_t k = 0; k < map->n; ++k) m.data[k] = map->data[k];
        if (m.n && (m.lo[0] != 0 || m.lo[m.n] != t->d.buckets))
            return fail(XPIR_EINVAL, "table_apply: shard map must cover every bucket");
    } else if (t->sharded()) {
        return fail(XPIR_EINVAL, "table_apply: a payload shard needs the shard map");
    }
    DeviceGuard g(t->device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : t->stream;
    XCK(t->gather.ensure(uint64_t(t->h.n_touched) * t->d.item));
    t->d.gather = t->gather.as<uint8_t>();
    XCK(launch_cuckoo_gather_sharded(t->d, &t->h, t->lo, t->hi, t->data, m, s));
    count_launches(1);
    if (!stream) XCK(cudaStreamSynchronize(s));
    return XPIR_OK;
}

int xpir_table_apply_scatter_dev(xpir_table* t, const uint8_t* d_payload, void* stream) {
    if (!t) return fail(XPIR_EINVAL, "table_apply: null table");
    if (t->h.n_touched && !d_payload) return fail(XPIR_EINVAL, "table_apply: null payload");
    DeviceGuard g(t->device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : t->stream;
    XCK(launch_cuckoo_scatter_sharded(t->d, &t->h, t->lo, t->hi, t->data, d_payload, s));
    count_launches(1);
    if (!stream) XCK(cudaStreamSynchronize(s));
    return XPIR_OK;
}

int xpir_table_shard(const xpir_table* t, uint32_t* lo, uint32_t* hi) {
    if (!t) return fail(XPIR_EINVAL, "table_shard: null table");
    if (lo) *lo = t->lo;
    if (hi) *hi = t->hi;
    return XPIR_OK;
}

int xpir_table_insert_batch(xpir_table* t, const uint32_t* b1, const uint32_t* b2,
                            const uint8_t* payload, uint64_t n, uint32_t* reports) {
    if (!t) return fail(XPIR_EINVAL, "table_insert: null table");
    if (n == 0) return XPIR_OK;
    if (!b1 || !b2 || !payload) return fail(XPIR_EINVAL, "table_insert: null buffer");
    // cuckoo.cpp:57-58 — validated per item in order; items before the bad one
    // are inserted, exactly as a loop of Table::insert calls would leave them.
    uint64_t ok = n;
    for (uint64_t k = 0; k < n; ++k)
        if (b1[k] >= t->d.buckets || b2[k] >= t->d.buckets) {
            ok = k;
            break;
        }
    std::lock_guard<std::mutex> lk(t->mu);
    DeviceGuard g(t->device);
    cudaStream_t s = t->stream;
    if (ok > 0) {
        XCK(t->in_b1.ensure(4 * ok));
        XCK(t->in_b2.ensure(4 * ok));
        XCK(t->in_payload.ensure(ok * t->d.item));
        XCK(t->in_reports.ensure(16 * ok));
        XCK(cudaMemcpyAsync(t->in_b1.p, b1, 4 * ok, cudaMemcpyHostToDevice, s));
        XCK(cudaMemcpyAsync(t->in_b2.p, b2, 4 * ok, cudaMemcpyHostToDevice, s));
        XCK(cudaMemcpyAsync(t->in_payload.p, payload, ok * t->d.item, cudaMemcpyHostToDevice, s));
        int rc = xpir_table_insert_batch_dev(t, t->in_b1.as<uint32_t>(), t->in_b2.as<uint32_t>(),
                                             t->in_payload.as<uint8_t>(), ok,
                                             t->in_reports.as<uint32_t>(), s);
        if (rc) return rc;
        if (reports)
            XCK(cudaMemcpyAsync(reports, t->in_reports.p, 16 * ok, cudaMemcpyDeviceToHost, s));
        XCK(cudaStreamSynchronize(s));
    }
    if (ok < n) return fail(XPIR_EINVAL, "cuckoo: bucket index out of range");
    return XPIR_OK;
}

int xpir_table_reserve(xpir_table* t, uint64_t max_batch) {
    if (!t) return fail(XPIR_EINVAL, "table_reserve: null table");
    std::lock_guard<std::mutex> lk(t->mu);
    DeviceGuard g(t->device);
    const uint64_t n = std::min<uint64_t>(max_batch, t->slots());
    XCK(t->gather.ensure(n * t->d.item));
    XCK(t->in_b1.ensure(4 * max_batch));
    XCK(t->in_b2.ensure(4 * max_batch));
    XCK(t->in_reports.ensure(16 * max_batch));
    XCK(cuckoo_reserve(t->par, max_batch, t->d.buckets, t->stream));  // claim-sort scratch
    XCK(cudaStreamSynchronize(t->stream));
    return XPIR_OK;
}

int xpir_table_snapshot(const xpir_table* t, uint8_t* host_out) {
    if (!t || !host_out) return fail(XPIR_EINVAL, "table_snapshot: null argument");
    DeviceGuard g(t->device);
    XCK(cudaStreamSynchronize(t->stream));
    XCK(cudaMemcpy(host_out, t->data, t->data_bytes(), cudaMemcpyDeviceToHost));
    return XPIR_OK;
}

void* xpir_table_device_data(const xpir_table* t) { return t ? t->data : nullptr; }

int xpir_table_seal(const xpir_table* t, xpir_store* st, uint64_t epoch, void* stream) {
    if (!t || !st) return fail(XPIR_EINVAL, "table_seal: null argument");
    if (st->N != t->d.buckets || uint64_t(st->S) != uint64_t(t->d.depth) * t->d.item)
        return fail(XPIR_EINVAL, "table_seal: store geometry differs from the table");
    if (st->device != t->device) return fail(XPIR_EINVAL, "table_seal: different devices");
    if (st->lo < t->lo || st->hi > t->hi) return fail(XPIR_EINVAL, "table_seal: store range outside the payload shard");
    DeviceGuard g(t->device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : t->stream;
    XCK(cudaMemcpyAsync(st->data, t->data + uint64_t(st->lo - t->lo) * st->S, st->bytes(),
                        cudaMemcpyDeviceToDevice, s));
    if (!stream) XCK(cudaStreamSynchronize(s));
    st->epoch = epoch;
    return XPIR_OK;
}

int xpir_table_meta(const xpir_table* t, uint8_t* used, uint32_t* b1, uint32_t* b2,
                    uint64_t* stamp) {
    if (!t) return fail(XPIR_EINVAL, "table_meta: null table");
    DeviceGuard g(t->device);
    XCK(cudaStreamSynchronize(t->stream));
    const uint64_t n = t->slots();
    if (used) XCK(cudaMemcpy(used, t->d.used, n, cudaMemcpyDeviceToHost));
    if (b1) XCK(cudaMemcpy(b1, t->d.beta1, 4 * n, cudaMemcpyDeviceToHost));
    if (b2) XCK(cudaMemcpy(b2, t->d.beta2, 4 * n, cudaMemcpyDeviceToHost));
    if (stamp) XCK(cudaMemcpy(stamp, t->d.stamp, 8 * n, cudaMemcpyDeviceToHost));
    return XPIR_OK;
}

int xpir_table_counters(const xpir_table* t, uint64_t* writes, uint64_t* live, uint64_t* next_stamp) {
    if (!t) return fail(XPIR_EINVAL, "table_counters: null table");
    if (writes) *writes = t->h.writes;
    if (live) *live = t->h.live;
    if (next_stamp) *next_stamp = t->h.next_stamp;
    return XPIR_OK;
}

int xpir_table_slot_used(const xpir_table* t, uint32_t bucket, uint32_t slot) {
    if (!t || bucket >= t->d.buckets || slot >= t->d.depth)
        return fail(XPIR_EINVAL, "slot_used: out of range");
    DeviceGuard g(t->device);
    uint8_t u = 0;
    XCK(cudaStreamSynchronize(t->stream));
    XCK(cudaMemcpy(&u, t->d.used + uint64_t(bucket) * t->d.depth + slot, 1, cudaMemcpyDeviceToHost));
    return u ? 1 : 0;
}

int xpir_table_state_digest(const xpir_table* t, uint8_t out[32]) {
    if (!t || !out) return fail(XPIR_EINVAL, "state_digest: null argument");
    if (t->sharded()) return fail(XPIR_EINVAL, "state_digest: needs the whole table (this is a payload shard)");
    const uint64_t n = t->slots();
    std::vector<uint8_t> data(n * t->d.item), used(n);
    std::vector<uint32_t> b1(n), b2(n);
    std::vector<uint64_t> st(n);
    int rc = xpir_table_snapshot(t, data.data());
    if (rc) return rc;
    rc = xpir_table_meta(t, used.data(), b1.data(), b2.data(), st.data());
    if (rc) return rc;
    HostBlake2b h(32);  // cuckoo.cpp:137-149
    h.update_u64be(t->h.writes);
    h.update_u64be(t->h.live);
    h.update_u64be(t->h.next_stamp);
    h.update(data.data(), data.size());
    for (uint64_t f = 0; f < n; ++f) {
        h.update_u64be(used[f] ? 1 : 0);
        h.update_u64be(uint64_t(b1[f]) << 32 | b2[f]);
        h.update_u64be(st[f]);
    }
    h.final(out);
    return XPIR_OK;
}

}  // extern "C"

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

struct xpir_window {
    int device;
    uint32_t m, h, w;
    uint64_t base = 0;
    uint64_t words;
    std::deque<unsigned long long*> deltas;
    cudaStream_t stream = nullptr;
    DevBuf pos, seqs, scratch, enc;
    std::mutex mu;
};

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
    if (e == cudaSuccess) e = cudaMemset(d, 0, 8 * win->words);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&win->stream, cudaStreamNonBlocking);
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
    unsigned long long* d = nullptr;
    XCK(cudaMalloc(&d, 8 * win->words));
    XCK(cudaMemsetAsync(d, 0, 8 * win->words, win->stream));
    win->deltas.push_back(d);
    while (win->deltas.size() > win->w) {
        XCK(cudaStreamSynchronize(win->stream));
        cudaFree(win->deltas.front());
        win->deltas.pop_front();
        win->base++;
    }
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

int xpir_window_digest(const xpir_window* win, uint8_t out[32]) {  // notify.cpp:87-107
    if (!win) return fail(XPIR_EINVAL, "window_digest: null argument");
    return xpir_window_digest_n(win, win->deltas.size(), out);
}

int xpir_window_digest_n(const xpir_window* win, uint64_t count, uint8_t out[32]) {  // Window::digest(count)
    if (!win || !out) return fail(XPIR_EINVAL, "window_digest: null argument");
    if (count > win->deltas.size()) return fail(XPIR_EINVAL, "Window::digest: count too large");  // notify.cpp:92
    HostBlake2b h(32);
    const char* tag = "interest-window-v1";
    h.update(reinterpret_cast<const uint8_t*>(tag), std::strlen(tag));
    h.update_u64be(win->m);
    h.update_u64be(win->h);
    h.update_u64be(win->w);
    h.update_u64be(win->base);
    h.update_u64be(count);
    std::vector<uint64_t> words(win->words);
    for (uint64_t i = 0; i < count; ++i) {
        int rc = xpir_window_delta(win, i, words.data());
        if (rc) return rc;
        h.update(reinterpret_cast<const uint8_t*>(words.data()), 8 * words.size());  // LE words
    }
    h.final(out);
    return XPIR_OK;
}

// notify::encode_delta (notify.cpp:131-149) of delta i (0 = oldest) on device.
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

// notify::decode_delta (notify.cpp:131-170). EINVAL = the reference's nullopt.
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

// ===========================================================================
// replica state machine — server::ServerCore (server.hpp:57-98, server.cpp:28-91)
// on device: cuckoo table + interest window + a ring of sealed stores.
// ===========================================================================
struct xpir_server {
    int device;
    xpir_table* table = nullptr;
    xpir_window* window = nullptr;
    uint32_t rotate_writes, epoch_ring;
    uint64_t writes = 0, latest_epoch = 0;
    struct Sealed {
        uint64_t epoch;
        uint32_t since_batch;  // table batch id the image is synchronised with
        xpir_store* st;
    };
    std::deque<Sealed> ring;  // oldest first
    std::mutex mu;
};

static int server_seal(xpir_server* sv, uint64_t* epoch_out) {  // server.cpp:75-81
    xpir_table* t = sv->table;
    DeviceGuard g(sv->device);
    xpir_server::Sealed e{};
    if (sv->ring.size() >= sv->epoch_ring) {
        // reuse the oldest image: only slots rewritten since it was sealed are copied
        e = sv->ring.front();
        sv->ring.pop_front();
        XCK(launch_seal_incremental(t->d, t->lo, t->hi, e.since_batch, t->data, e.st->data, num_sms(sv->device),
                                    t->stream));
        count_launches(1);
    } else {
        int rc = xpir_store_create(sv->device, t->d.buckets, uint32_t(t->d.depth * t->d.item), t->lo, t->hi, &e.st);
        if (rc) return rc;
        XCK(cudaMemcpyAsync(e.st->data, t->data, e.st->bytes(), cudaMemcpyDeviceToDevice, t->stream));
    }
    XCK(cudaStreamSynchronize(t->stream));
    e.since_batch = t->h.batch_id;
    e.epoch = ++sv->latest_epoch;
    e.st->epoch = e.epoch;
    sv->ring.push_back(e);
    if (epoch_out) *epoch_out = e.epoch;
    return XPIR_OK;
}

extern "C" {

int xpir_server_create(int device, uint32_t buckets, uint32_t depth, uint64_t capacity, uint64_t item_size,
                       const uint8_t seed[32], uint32_t m_bits, uint32_t h, uint32_t window_deltas,
                       uint32_t rotate_writes, uint32_t epoch_ring, xpir_server** out) {
    return xpir_server_create_shard(device, buckets, depth, capacity, item_size, seed, m_bits, h, window_deltas,
                                    rotate_writes, epoch_ring, 0, buckets, out);
}

int xpir_server_create_shard(int device, uint32_t buckets, uint32_t depth, uint64_t capacity, uint64_t item_size,
                             const uint8_t seed[32], uint32_t m_bits, uint32_t h, uint32_t window_deltas,
                             uint32_t rotate_writes, uint32_t epoch_ring, uint32_t lo, uint32_t hi,
                             xpir_server** out) {
    if (!out) return fail(XPIR_EINVAL, "server_create: null out");
    if (rotate_writes == 0) return fail(XPIR_EINVAL, "server_create: rotate_writes must be positive");
    if (epoch_ring == 0) return fail(XPIR_EINVAL, "server_create: epoch_ring must be positive");
    auto* sv = new xpir_server;
    sv->device = device;
    sv->rotate_writes = rotate_writes;
    sv->epoch_ring = epoch_ring;
    int rc = xpir_table_create_shard(device, buckets, depth, capacity, item_size, seed, lo, hi, &sv->table);
    if (!rc) rc = xpir_window_create(device, m_bits, h, window_deltas, &sv->window);
    if (!rc) rc = xpir_window_rotate(sv->window);  // server.cpp:40
    if (!rc) rc = server_seal(sv, nullptr);          // server.cpp:42, epoch 1 (all zeros)
    if (rc) {
        std::string msg = g_err;
        xpir_server_destroy(sv);
        return fail(rc, msg);
    }
    *out = sv;
    return XPIR_OK;
}

int xpir_server_destroy(xpir_server* sv) {
    if (!sv) return XPIR_OK;
    for (auto& e : sv->ring) xpir_store_destroy(e.st);
    xpir_table_destroy(sv->table);
    xpir_window_destroy(sv->window);
    delete sv;
    return XPIR_OK;
}

int xpir_server_apply_round(xpir_server* sv, const uint32_t* beta1, const uint32_t* beta2, const uint8_t* payload,
                            const uint32_t* interest, uint32_t h_per_write, uint64_t n, int seal_after,
                            uint32_t* reports, uint64_t* sealed_epoch) {
    return xpir_server_apply_round_sharded(sv, beta1, beta2, payload, interest, h_per_write, n, seal_after, nullptr,
                                           nullptr, nullptr, reports, sealed_epoch);
}

// The table insert of a round on a payload shard: H2D, replicated walk, gather
// (peer shards), the caller's barrier, scatter.
static int table_insert_sharded(xpir_table* t, const uint32_t* b1, const uint32_t* b2, const uint8_t* payload,
                                uint64_t n, uint32_t* reports, const xpir_shard_map* map,
                                void (*barrier)(void*), void* ctx) {
    std::lock_guard<std::mutex> lk(t->mu);
    DeviceGuard g(t->device);
    cudaStream_t s = t->stream;
    XCK(t->in_b1.ensure(4 * n));
    XCK(t->in_b2.ensure(4 * n));
    XCK(t->in_payload.ensure(n * t->d.item));
    XCK(t->in_reports.ensure(16 * n));
    XCK(cudaMemcpyAsync(t->in_b1.p, b1, 4 * n, cudaMemcpyHostToDevice, s));
    XCK(cudaMemcpyAsync(t->in_b2.p, b2, 4 * n, cudaMemcpyHostToDevice, s));
    XCK(cudaMemcpyAsync(t->in_payload.p, payload, n * t->d.item, cudaMemcpyHostToDevice, s));
    int rc = xpir_table_insert_walk_dev(t, t->in_b1.as<uint32_t>(), t->in_b2.as<uint32_t>(), n,
                                        t->in_reports.as<uint32_t>(), s);
    if (!rc) rc = xpir_table_apply_gather_dev(t, map, s);
    if (rc) return rc;
    XCK(cudaStreamSynchronize(s));
    if (barrier) barrier(ctx);  // every shard has staged what moves into its range
    rc = xpir_table_apply_scatter_dev(t, t->in_payload.as<uint8_t>(), s);
    if (rc) return rc;
    if (reports) XCK(cudaMemcpyAsync(reports, t->in_reports.p, 16 * n, cudaMemcpyDeviceToHost, s));
    XCK(cudaStreamSynchronize(s));
    return XPIR_OK;
}

int xpir_server_apply_round_sharded(xpir_server* sv, const uint32_t* beta1, const uint32_t* beta2,
                                    const uint8_t* payload, const uint32_t* interest, uint32_t h_per_write,
                                    uint64_t n, int seal_after, const xpir_shard_map* map,
                                    void (*barrier)(void*), void* barrier_ctx, uint32_t* reports,
                                    uint64_t* sealed_epoch) {
    if (!sv) return fail(XPIR_EINVAL, "server_apply: null server");
    if (sv->table->sharded() && (!map || !barrier))
        return fail(XPIR_EINVAL, "server_apply: a payload shard needs the shard map and a barrier");
    if (sealed_epoch) *sealed_epoch = 0;
    if (n && (!beta1 || !beta2 || !payload || (h_per_write && !interest)))
        return fail(XPIR_EINVAL, "server_apply: null buffer");
    std::lock_guard<std::mutex> lk(sv->mu);
    // apply_write (server.cpp:58-73) for writes in order: beta range check
    // (server.cpp:60-61) happens before any state changes of that write.
    uint64_t ok = n;
    for (uint64_t k = 0; k < n; ++k)
        if (beta1[k] >= sv->table->d.buckets || beta2[k] >= sv->table->d.buckets) {
            ok = k;
            break;
        }
    if (ok) {
        int rc = sv->table->sharded()
                     ? table_insert_sharded(sv->table, beta1, beta2, payload, ok, reports, map, barrier, barrier_ctx)
                     : xpir_table_insert_batch(sv->table, beta1, beta2, payload, ok, reports);
        if (rc) return rc;
        // interest positions per rotation segment, then rotate (server.cpp:64-70)
        uint64_t a = 0;
        while (a < ok) {
            const uint64_t to_rot = sv->rotate_writes - (sv->writes % sv->rotate_writes);
            const uint64_t b = std::min(ok, a + to_rot);
            if (h_per_write) {
                rc = xpir_window_absorb(sv->window, interest + a * h_per_write, (b - a) * h_per_write);
                if (rc) return rc;
            }
            sv->writes += b - a;
            if (sv->writes % sv->rotate_writes == 0) {
                rc = xpir_window_rotate(sv->window);
                if (rc) return rc;
            }
            a = b;
        }
    }
    if (ok < n) return fail(XPIR_EINVAL, "write targets a bucket outside the table");
    if (seal_after) return server_seal(sv, sealed_epoch);
    return XPIR_OK;
}

int xpir_server_seal(xpir_server* sv, uint64_t* epoch) {
    if (!sv) return fail(XPIR_EINVAL, "server_seal: null server");
    std::lock_guard<std::mutex> lk(sv->mu);
    return server_seal(sv, epoch);
}

int xpir_server_snapshot(xpir_server* sv, uint64_t epoch, xpir_store** st) {  // server.cpp:83-91
    if (!sv || !st) return fail(XPIR_EINVAL, "server_snapshot: null argument");
    std::lock_guard<std::mutex> lk(sv->mu);
    *st = nullptr;
    if (epoch == 0) epoch = sv->latest_epoch;
    for (auto& e : sv->ring)
        if (e.epoch == epoch) *st = e.st;
    return *st ? XPIR_OK : fail(XPIR_EINVAL, "server_snapshot: epoch not in the ring");
}

// ServerCore::make_freeze (server.cpp:45-56): the deltas that will never change
// again (all but the newest) — base, newest index, digest over them, and their
// count; delta k's wire bytes come from xpir_window_encode_delta(window, k, ...).
int xpir_server_freeze(xpir_server* sv, uint64_t* base, uint64_t* newest, uint8_t digest[32], uint64_t* count) {
    if (!sv || !base || !newest || !digest || !count) return fail(XPIR_EINVAL, "server_freeze: null argument");
    std::lock_guard<std::mutex> lk(sv->mu);
    xpir_window* w = sv->window;
    const uint64_t size = w->deltas.size();
    *base = w->base;
    *newest = w->base + size - 2;  // window.newest() - 1
    *count = size - 1;
    return xpir_window_digest_n(w, size - 1, digest);
}

int xpir_server_info(xpir_server* sv, uint64_t* writes, uint64_t* latest_epoch, uint64_t* oldest_epoch,
                     xpir_table** table, xpir_window** window) {
    if (!sv) return fail(XPIR_EINVAL, "server_info: null server");
    std::lock_guard<std::mutex> lk(sv->mu);
    if (writes) *writes = sv->writes;
    if (latest_epoch) *latest_epoch = sv->latest_epoch;
    if (oldest_epoch) *oldest_epoch = sv->ring.empty() ? 0 : sv->ring.front().epoch;
    if (table) *table = sv->table;
    if (window) *window = sv->window;
    return XPIR_OK;
}

}  // extern "C"
