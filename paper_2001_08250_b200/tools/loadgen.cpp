// Host load generator for the read path (bench_batcher.py): T native threads
// issue single masked requests back to back, as node.cpp's session and link
// threads call server::answer_share (node.cpp:263-266, 528-530), either through
// the read batcher (mode 0: xpir_batcher_answer) or one scan per request
// (mode 1: xpir_answer_batch with B = 1). Benchmark tooling, not product code.
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <string>
#include <thread>
#include <vector>

#include "../../include/xpir.h"

extern "C" int xpl_drive(int mode, void* target, uint32_t N, uint32_t S, const uint8_t* qpool, uint32_t pool,
                         const uint8_t* seeds, uint32_t threads, double seconds, double warm, double* rate,
                         char* err, uint32_t err_len) {
    const size_t nb = (N + 7) / 8;
    std::atomic<bool> stop{false}, counting{false};
    std::atomic<int> first_rc{0};
    std::vector<uint64_t> counts(threads, 0);
    std::string msg;
    std::vector<std::thread> ts;
    for (uint32_t t = 0; t < threads; ++t)
        ts.emplace_back([&, t] {
            std::vector<uint8_t> out(S);
            for (uint64_t i = 0; !stop.load(std::memory_order_relaxed); ++i) {
                const uint32_t k = uint32_t((uint64_t(t) * 7919 + i) % pool);
                const int rc = mode == 0
                                   ? xpir_batcher_answer(static_cast<xpir_batcher*>(target), qpool + k * nb, N,
                                                         seeds + size_t(k) * 32, out.data())
                                   : xpir_answer_batch(static_cast<xpir_store*>(target), qpool + k * nb, nb, N, 1,
                                                       seeds + size_t(k) * 32, out.data());
                if (rc) {
                    int z = 0;
                    if (first_rc.compare_exchange_strong(z, rc)) msg = xpir_last_error();
                    stop = true;
                    break;
                }
                if (counting.load(std::memory_order_relaxed)) counts[t]++;
            }
        });
    std::this_thread::sleep_for(std::chrono::duration<double>(warm));
    counting = true;
    const auto t0 = std::chrono::steady_clock::now();
    std::this_thread::sleep_for(std::chrono::duration<double>(seconds));
    uint64_t n = 0;
    for (uint64_t c : counts) n += c;
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    stop = true;
    for (auto& th : ts) th.join();
    *rate = double(n) / dt;
    if (first_rc && err && err_len) {
        std::snprintf(err, err_len, "%s", msg.c_str());
    }
    return first_rc;
}
