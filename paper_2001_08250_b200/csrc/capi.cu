// extern "C" boundary (include/xpir.h) over the sm_100a kernels: the core —
// errors, scan options and timing, device/IPC helpers, the sealed-snapshot
// store and the scan dispatch, the primitives. The cuckoo table, the interest
// window and the device ServerCore are in capi_table.cu, capi_window.cu and
// capi_server.cu. Host-side bookkeeping only: argument validation with the
// reference's error conditions, device memory ownership, kernel dispatch.
// There is no CPU compute path: every answer, table mutation and filter update
// is produced by a kernel, and the library fails (XPIR_ECUDA) without a GPU.
#include "capi_internal.cuh"

namespace xpir {
static std::atomic<uint64_t> g_launches{0};
void count_launches(uint64_t n) { g_launches += n; }
namespace capi {
thread_local std::string g_err;
std::atomic<int> g_last_kernel{0};
xpir_scan_opts g_opts{};
std::mutex g_opts_mu;
int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}
const std::string& last_error_message() { return g_err; }
}  // namespace capi
int set_error(int code, const std::string& msg) { return capi::fail(code, msg); }
// Drop the per-stream query scratch of `s` (its owner is destroying the stream;
// all work on it has completed).
void store_release_stream_scratch(xpir_store* st, cudaStream_t s) {
    if (!st) return;
    std::lock_guard<std::mutex> lk(st->scratch_mu);
    for (auto it = st->qwin_by_stream.begin(); it != st->qwin_by_stream.end(); ++it)
        if (it->first == s) {
            it->second->release();
            delete it->second;
            st->qwin_by_stream.erase(it);
            return;
        }
}
}  // namespace xpir

// ===========================================================================
// store
// ===========================================================================

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

int xpir_set_host_sync(int mode) {
    static const unsigned flags[4] = {cudaDeviceScheduleAuto, cudaDeviceScheduleSpin, cudaDeviceScheduleYield,
                                      cudaDeviceScheduleBlockingSync};
    if (mode < 0 || mode > 3) return fail(XPIR_EINVAL, "set_host_sync: mode 0..3");
    set_sync_flags(flags[mode]);
    return XPIR_OK;
}

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

// Per-thread, per-device scratch of the small host-buffer entry points
// (mask_answer, prng_expand, prf_batch, make_interest_batch, bloom_positions):
// a grow-only device buffer and a non-blocking stream, so a call is
// copy-in / kernel / copy-out / stream sync — no cudaMalloc/cudaFree (cudaFree
// synchronises the whole device, stalling every concurrent scan) and no work on
// the legacy default stream.
struct CallScratch {
    int device = -1;
    cudaStream_t s = nullptr;
    DevBuf dev;
    ~CallScratch() {
        if (s) cudaStreamDestroy(s);
        dev.release();
    }
};
CallScratch& call_scratch() {
    thread_local CallScratch per_dev[16];
    int d = 0;
    cudaGetDevice(&d);
    CallScratch& cs = per_dev[d & 15];
    if (cs.device != d) {
        if (cs.s) cudaStreamDestroy(cs.s);
        cs.dev.release();
        cs.s = nullptr;
        cs.device = d;
        if (cudaStreamCreateWithFlags(&cs.s, cudaStreamNonBlocking) != cudaSuccess) cs.s = nullptr;
    }
    return cs;
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
    st->peer_partial.release();
    st->peer_cnt.release();
    st->peer_stats.release();
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
// Batch-size crossovers from the config-5 sweep: below 24 the direct
// kernel, nibble tables (7) from 24, 6-bucket tables (9) for 129..256 (6-15% faster
// than the nibble tables there: 1 GiB store, S = 1024/4096, B = 256 1.96 vs 2.30 ms;
// past 256 its request tiles split), byte tables (2/5) from 257, 9-bucket quad tables (8) or
// half-TMEM byte tables (5) by the calibrated cost model from 2048.
static const uint32_t g_k4_min_batch = 24;
static const uint32_t g_k6_min_batch = 129, g_k6_max_batch = 256;
static const uint32_t g_m4_min_batch = 257;
static const uint32_t g_q_min_batch = 2048;

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
        k = !m4_ok ? 1
            : (B >= g_k6_min_batch && B <= g_k6_max_batch) ? 9
            : B >= g_m4_min_batch ? 2 : B >= g_k4_min_batch ? 7 : 1;
    }
    if (k == 6) k = 1;  // (the warp-private nibble kernel was retired in round 2)
    if ((k == 2 || k == 7 || k == 9) && !m4_ok) k = 1;
    if ((k == 8 ) && !q_ok) k = 1;
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
    if (kernel == 8) {  // quad-interleaved 9-bucket tables, full-TMEM accumulators
        timing_begin(s, &ev);
        XCK(launch_scan_m4rm_q(a, num_sms(st->device)));
        timing_end(s, ev);
        count_launches(1);
        g_last_kernel = 8;
        return XPIR_OK;
    }
    if (kernel == 9) {  // 6-bucket tables
        timing_begin(s, &ev);
        XCK(launch_scan_m4rm6(a, num_sms(st->device)));
        timing_end(s, ev);
        count_launches(1);
        g_last_kernel = 9;
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
    if (k != 2 && k != 7 && k != 8 && k != 9) return run_rows(st, k, rows + blo, stride, B, d_out, s);
    const uint64_t qs = m4rm_qstride(B);
    DevBuf& qw = st->qwin_for(s);
    XCK(qw.ensure(m4rm_qrows(nbw) * qs));
    XCK(launch_transpose_q(rows, stride, blo, nbw, B, qw.as<uint8_t>(), qs, s, m4rm_layout(k)));
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
    if (k == 2 || k == 7 || k == 8 || k == 9) {
        const uint64_t qs = m4rm_qstride(B);
        DevBuf& qw = st->qwin_for(s);
        XCK(qw.ensure(m4rm_qrows(nbw) * qs));
        XCK(launch_expand_T(d_seeds, B, blo, nbw, qw.as<uint8_t>(), qs, s, m4rm_layout(k)));
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
    if (k == 2 || k == 7 || k == 8 || k == 9) {
        const uint64_t qs = m4rm_qstride(B);
        XCK(st->qwin.ensure(m4rm_qrows(nbw) * qs));
        XCK(launch_transpose_q(st->q.as<uint8_t>(), ws, 0, nbw, B, st->qwin.as<uint8_t>(), qs, s, m4rm_layout(k)));
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
    if (k == 2 || k == 7 || k == 8 || k == 9) {
        const uint64_t qs = m4rm_qstride(B);
        XCK(st->qwin.ensure(m4rm_qrows(nbw) * qs));
        XCK(launch_transpose_q(st->q.as<uint8_t>(), ws, 0, nbw, B, st->qwin.as<uint8_t>(), qs, s, m4rm_layout(k)));
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
                                      uint32_t self_rank, void* stream) {
    if (!st) return fail(XPIR_EINVAL, "answer_batch_seeded_peer: null store");
    if (n_ranks < 1 || n_ranks > 8) return fail(XPIR_EINVAL, "answer_batch_seeded_peer: 1..8 ranks");
    if (self_rank >= n_ranks) return fail(XPIR_EINVAL, "answer_batch_seeded_peer: self_rank out of range");
    if (!out_ptrs || !row_bounds || (B && !d_seeds)) return fail(XPIR_EINVAL, "answer_batch_seeded_peer: null");
    if (row_bounds[0] != 0 || row_bounds[n_ranks] != B)
        return fail(XPIR_EINVAL, "answer_batch_seeded_peer: row bounds must cover [0, B)");
    if (st->S % 32 != 0 || B < 2048)
        return fail(XPIR_EINVAL, "answer_batch_seeded_peer: fused reduce needs S % 32 == 0 and B >= 2048");
    DeviceGuard g(st->device);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : st->stream;
    const uint64_t blo = st->byte_lo(), nbw = st->nbytes_window();
    const uint64_t qs = m4rm_qstride(B);
    // fix-up state of the fused epilogue: zero at (re)allocation, kept zero by the kernel
    const uint64_t tiles = uint64_t(st->S / 32) * ((B + 2047) / 2048);
    auto zeroed = [&](DevBuf& b, uint64_t n) -> cudaError_t {
        const size_t cap0 = b.cap;
        const void* p0 = b.p;
        cudaError_t e = b.ensure(n);
        if (e == cudaSuccess && (b.cap != cap0 || b.p != p0)) e = cudaMemsetAsync(b.p, 0, b.cap, s);
        return e;
    };
    XCK(zeroed(st->peer_partial, uint64_t(B) * st->S));
    XCK(zeroed(st->peer_cnt, 4 * tiles));
    XCK(zeroed(st->peer_stats, 16));
    DevBuf& qw = st->qwin_for(s);
    XCK(qw.ensure(m4rm_qrows(nbw) * qs));
    XCK(launch_expand_T(d_seeds, B, blo, nbw, qw.as<uint8_t>(), qs, s, m4rm_layout(8)));  // the fused path always runs kernel 8
    M4Args a{st->data, st->nb(), st->S, qw.as<uint8_t>(), qs, B, out_ptrs[0], s};
    a.peers.n = n_ranks;
    a.peers.self = self_rank;
    for (uint32_t k = 0; k < n_ranks; ++k) {
        a.peers.ptr[k] = out_ptrs[k];
        a.peers.bound[k] = row_bounds[k];
    }
    a.peers.bound[n_ranks] = row_bounds[n_ranks];
    a.peers.partial = st->peer_partial.as<uint8_t>();
    a.peers.tile_cnt = st->peer_cnt.as<uint32_t>();
    a.peers.stats = st->peer_stats.as<unsigned long long>();
    cudaEvent_t ev;
    timing_begin(s, &ev);
    XCK(launch_scan_m4rm_q(a, num_sms(st->device)));
    timing_end(s, ev);
    count_launches(2);
    g_last_kernel = 8;
    return XPIR_OK;
}

int xpir_store_peer_stats(xpir_store* st, uint64_t* remote_bytes, uint64_t* own_bytes, int reset) {
    if (!st) return fail(XPIR_EINVAL, "store_peer_stats: null store");
    uint64_t v[2] = {0, 0};
    if (st->peer_stats.p) {
        DeviceGuard g(st->device);
        XCK(cudaDeviceSynchronize());
        XCK(cudaMemcpy(v, st->peer_stats.p, 16, cudaMemcpyDeviceToHost));
        if (reset) {
            XCK(cudaMemset(st->peer_stats.p, 0, 16));
            XCK(cudaDeviceSynchronize());
        }
    }
    if (remote_bytes) *remote_bytes = v[0];
    if (own_bytes) *own_bytes = v[1];
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
    CallScratch& cs = call_scratch();
    if (!cs.s) return fail(XPIR_ECUDA, "mask_answer: no stream");
    XCK(cs.dev.ensure(len + 32));
    uint8_t* d = cs.dev.as<uint8_t>();
    XCK(cudaMemcpyAsync(d, ans, len, cudaMemcpyHostToDevice, cs.s));
    XCK(cudaMemcpyAsync(d + len, seed, 32, cudaMemcpyHostToDevice, cs.s));
    // one "request" of S = len bytes: out = ans ^ pad
    XCK(launch_init_out(d, 1, uint32_t(len), d + len, true, cs.s));
    count_launches(1);
    XCK(cudaMemcpyAsync(out, d, len, cudaMemcpyDeviceToHost, cs.s));
    XCK(cudaStreamSynchronize(cs.s));
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
    CallScratch& cs = call_scratch();
    if (!cs.s) return fail(XPIR_ECUDA, "prng_expand: no stream");
    XCK(cs.dev.ensure(len));
    XCK(launch_keystream(seed, 0, 0, cs.dev.as<uint8_t>(), len, cs.s));
    count_launches(1);
    XCK(cudaMemcpyAsync(out, cs.dev.p, len, cudaMemcpyDeviceToHost, cs.s));
    XCK(cudaStreamSynchronize(cs.s));
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
    CallScratch& cs = call_scratch();
    if (!cs.s) return fail(XPIR_ECUDA, "prf: no stream");
    XCK(cs.dev.ensure(16 * n));
    uint64_t* d = cs.dev.as<uint64_t>();
    XCK(cudaMemcpyAsync(d, inputs, 8 * n, cudaMemcpyHostToDevice, cs.s));
    XCK(launch_prf(ld64le(key), ld64le(key + 8), d, n, modulus, d + n, nullptr, cs.s));
    count_launches(1);
    XCK(cudaMemcpyAsync(out, d + n, 8 * n, cudaMemcpyDeviceToHost, cs.s));
    XCK(cudaStreamSynchronize(cs.s));
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

int xpir_write_betas_dev(int device, const uint8_t k1[16], const uint8_t k2[16], const uint64_t* d_keys, uint64_t n,
                         uint32_t buckets, uint32_t* d_beta1, uint32_t* d_beta2, void* stream) {
    if (buckets == 0) return fail(XPIR_EINVAL, "prf: modulus must be positive");
    if (!k1 || !k2 || (n && (!d_keys || !d_beta1 || !d_beta2))) return fail(XPIR_EINVAL, "write_betas: null buffer");
    DeviceGuard g(device);
    const uint64_t a[2] = {ld64le(k1), ld64le(k1 + 8)}, c[2] = {ld64le(k2), ld64le(k2 + 8)};
    XCK(launch_prf2(a, c, d_keys, n, buckets, d_beta1, d_beta2, static_cast<cudaStream_t>(stream)));
    count_launches(1);
    return XPIR_OK;
}

int xpir_make_interest_batch(uint32_t m_bits, uint32_t h, const uint8_t id[16],
                             const uint64_t* seqs, uint64_t n, uint32_t* out) {
    if (m_bits == 0) return fail(XPIR_EINVAL, "bloom_positions: m_bits must be positive");
    if (!id || (n && (!seqs || !out))) return fail(XPIR_EINVAL, "make_interest: null buffer");
    if (!n || !h) return XPIR_OK;
    CallScratch& cs = call_scratch();
    if (!cs.s) return fail(XPIR_ECUDA, "make_interest: no stream");
    const uint64_t pos_off = round16(8 * n);
    XCK(cs.dev.ensure(pos_off + 4 * n * h));
    uint64_t* ds = cs.dev.as<uint64_t>();
    uint32_t* dp = reinterpret_cast<uint32_t*>(cs.dev.as<uint8_t>() + pos_off);
    XCK(cudaMemcpyAsync(ds, seqs, 8 * n, cudaMemcpyHostToDevice, cs.s));
    XCK(launch_interest(id, ds, n, h, m_bits, dp, nullptr, cs.s));
    count_launches(1);
    XCK(cudaMemcpyAsync(out, dp, 4 * n * h, cudaMemcpyDeviceToHost, cs.s));
    XCK(cudaStreamSynchronize(cs.s));
    return XPIR_OK;
}

int xpir_bloom_positions(const uint8_t* item, uint64_t len, uint32_t h, uint32_t m_bits,
                         uint32_t* out) {
    if (m_bits == 0) return fail(XPIR_EINVAL, "bloom_positions: m_bits must be positive");
    if (len > 120) return fail(XPIR_EINVAL, "bloom_positions: device port takes items <= 120 bytes");
    if ((len && !item) || (h && !out)) return fail(XPIR_EINVAL, "bloom_positions: null buffer");
    if (!h) return XPIR_OK;
    CallScratch& cs = call_scratch();
    if (!cs.s) return fail(XPIR_ECUDA, "bloom_positions: no stream");
    XCK(cs.dev.ensure(128 + 4 * uint64_t(h)));
    uint8_t* d = cs.dev.as<uint8_t>();
    if (len) XCK(cudaMemcpyAsync(d, item, len, cudaMemcpyHostToDevice, cs.s));
    uint32_t* dp = reinterpret_cast<uint32_t*>(d + 128);
    XCK(launch_bloom_item(d, uint32_t(len), h, m_bits, dp, cs.s));
    count_launches(1);
    XCK(cudaMemcpyAsync(out, dp, 4 * uint64_t(h), cudaMemcpyDeviceToHost, cs.s));
    XCK(cudaStreamSynchronize(cs.s));
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
