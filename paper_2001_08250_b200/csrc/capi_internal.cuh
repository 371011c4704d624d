// Internal header of the C-ABI TUs (capi*.cu): shared host helpers and the
// handle structs behind include/xpir.h. Not part of the public interface.
#pragma once
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
void count_launches(uint64_t n);
int set_error(int code, const std::string& msg);
namespace capi {
int fail(int code, const std::string& msg);   // sets the thread's xpir_last_error()
const std::string& last_error_message();
extern std::atomic<int> g_last_kernel;
extern xpir_scan_opts g_opts;
extern std::mutex g_opts_mu;
}  // namespace capi
}  // namespace xpir

using namespace xpir;
using xpir::capi::fail;

namespace xpir {
namespace capi {

#define XCK(expr)                                                                       \
    do {                                                                                \
        cudaError_t e_ = (expr);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return fail(XPIR_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// Host wait policy for this process's CUDA contexts (xpir_set_host_sync; the
// environment variable XPIR_SYNC = spin | yield | blocking applies it once, at
// the library's first device call).
inline void set_sync_flags(unsigned f) {
    int n = 0, cur = 0;
    cudaGetDeviceCount(&n);
    cudaGetDevice(&cur);
    for (int d = 0; d < n; ++d) {
        cudaSetDevice(d);
        cudaSetDeviceFlags(f);
    }
    cudaSetDevice(cur);
    cudaGetLastError();
}
inline bool apply_sync_policy() {
    const char* e = getenv("XPIR_SYNC");
    if (!e) return false;
    set_sync_flags(!strcmp(e, "blocking") ? cudaDeviceScheduleBlockingSync
                   : !strcmp(e, "yield")  ? cudaDeviceScheduleYield
                   : !strcmp(e, "spin")   ? cudaDeviceScheduleSpin
                                          : cudaDeviceScheduleAuto);
    return true;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        static const bool policy = apply_sync_policy();
        (void)policy;
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

inline int num_sms(int dev) {
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
    // grows geometrically (x1.5): a buffer sized by a per-round count that creeps
    // up (e.g. touched slots) is reallocated O(log) times, not every round —
    // cudaFree/cudaMalloc inside a round can stall for milliseconds or more
    cudaError_t ensure(size_t n) {
        if (n <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        size_t want = std::max({n, size_t(256), cap + cap / 2});
        cap = 0;
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

inline uint64_t round16(uint64_t x) { return (x + 15) & ~uint64_t(15); }

// Grow-only pinned host staging buffer. A caller packs host inputs into it and
// issues ONE async H2D copy; `ready` (recorded after the copies that read it)
// guards the next reuse, so no stream synchronisation is needed in between.
struct PinnedBuf {
    uint8_t* p = nullptr;
    size_t cap = 0;
    cudaEvent_t ready = nullptr;
    cudaError_t ensure(size_t n) {  // waits for the previous user of the buffer
        if (ready) {
            cudaError_t e = cudaEventSynchronize(ready);
            if (e != cudaSuccess) return e;
        } else {
            cudaError_t e = cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
            if (e != cudaSuccess) return e;
        }
        if (n <= cap) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        const size_t want = std::max({n, size_t(4096), cap + cap / 2});
        cap = 0;
        cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&p), want, cudaHostAllocPortable);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    cudaError_t release_after(cudaStream_t s) { return ready ? cudaEventRecord(ready, s) : cudaSuccess; }
    void release() {
        if (ready) cudaEventSynchronize(ready);
        if (p) cudaFreeHost(p);
        if (ready) cudaEventDestroy(ready);
        p = nullptr;
        cap = 0;
        ready = nullptr;
    }
};

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

}  // namespace capi
}  // namespace xpir
using namespace xpir::capi;

// ---- handle structs ------------------------------------------------------
struct xpir_store {
    int device;
    uint32_t N, S, lo, hi;
    uint64_t epoch = 0;
    uint8_t* data = nullptr;
    cudaStream_t stream = nullptr;
    DevBuf q, out, seeds, masks, qwin, qx, idx;
    DevBuf peer_partial, peer_cnt, peer_stats;  // fused cross-GPU epilogue (xpir_answer_batch_seeded_peer_dev)
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

struct xpir_table {
    int device;
    uint8_t seed[32];
    CuckooDev d{};
    CuckooState h{};
    CuckooState* dstate = nullptr;
    uint8_t* data = nullptr;  // payloads of buckets [lo, hi)
    uint32_t lo = 0, hi = 0;  // a payload shard of the logical table (metadata is whole)
    cudaStream_t stream = nullptr;
    DevBuf in_b1, in_b2, in_payload, in_reports, gather, chk, in_pack;
    PinnedBuf stage;              // host inputs of xpir_table_insert_batch, packed for one H2D
    PinnedBuf state_h;            // pinned mirror of the walk state (async H2D / D2H)
    cudaGraphExec_t g1 = nullptr; // one host write as a graph (xpir_table_insert_batch, n = 1)
    PinnedBuf g1_stage;           // its packed write + report, pinned
    DevBuf g1_dev;                //   and on device
    bool walked = false;          // a walk kernel ran this batch (pre-existing items may have moved)
    bool async_pending = false;   // xpir_table_insert_batch_async issued, xpir_table_finish not yet called
    struct {
        const uint32_t *b1, *b2;
        const uint8_t* payload;
        uint32_t* reports;
        uint64_t n;
        cudaStream_t s;
    } async{};
    bool state_on_device = false; // the walk of the current call ran without a host round trip:
    uint32_t max_touched = 0;     //   h is stale, n_touched <= max_touched until synced
    CuckooParScratch par;
    bool parallel_prefix = true;  // XPIR_CUCKOO_SEQUENTIAL=1 disables (A/B checks)
    std::mutex mu;
    uint64_t slots() const { return uint64_t(d.buckets) * d.depth; }
    uint64_t data_bytes() const { return uint64_t(hi - lo) * d.depth * d.item; }
    bool sharded() const { return lo != 0 || hi != d.buckets; }
};

// xpir_table_insert_walk_dev without the device-side bucket range check, for
// callers that validated beta1/beta2 on the host (capi_table.cu).
int table_walk_impl(xpir_table* t, const uint32_t* d_b1, const uint32_t* d_b2, uint64_t n, uint32_t* d_reports,
                    void* stream);

struct xpir_window {
    int device;
    uint32_t m, h, w;
    uint64_t base = 0;
    uint64_t words;
    std::deque<unsigned long long*> deltas;
    cudaStream_t stream = nullptr;
    DevBuf pos, seqs, scratch, enc;
    PinnedBuf stage;           // host positions of xpir_window_absorb_prechecked
    mutable PinnedBuf dstage;  // deltas staged for a digest (xpir_window_digest_n)
    mutable std::mutex mu;
};

// Window::absorb of positions already checked against m_bits on the host: one
// packed H2D + the OR kernel on the window's stream, no host round trip.
int window_absorb_prechecked(xpir_window* win, const uint32_t* pos, uint64_t n);

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
        uint32_t pins = 0;     // readers holding the image (xpir_server_snapshot_acquire)
    };
    std::deque<Sealed> ring;           // oldest first
    std::vector<Sealed> retired;       // left the ring while pinned; back to spare on the last release
    std::vector<xpir_store*> spare;    // images with no epoch (xpir_server_reserve, released retirees)
    std::mutex mu;
};

