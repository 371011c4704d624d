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

// Open loop: `threads` callers issue requests at a fixed aggregate rate (each
// thread on its own evenly spaced schedule, staggered), through the batcher
// (mode 0) or one scan per request (mode 1). Latency = completion time minus the
// scheduled issue time (queueing behind a late schedule included). Writes the
// achieved rate and the p50/p90/p99/max latency in microseconds.
#include <algorithm>
extern "C" int xpl_open_loop(int mode, void* target, uint32_t N, uint32_t S, const uint8_t* qpool, uint32_t pool,
                             const uint8_t* seeds, uint32_t threads, double rate, double seconds, double* out6) {
    using clk = std::chrono::steady_clock;
    const size_t nb = (N + 7) / 8;
    const double per_thread = rate / threads;
    const uint64_t n_each = uint64_t(per_thread * seconds);
    std::vector<std::vector<double>> lat(threads);
    std::atomic<int> first_rc{0};
    const auto t0 = clk::now() + std::chrono::milliseconds(50);
    std::vector<std::thread> ts;
    for (uint32_t t = 0; t < threads; ++t)
        ts.emplace_back([&, t] {
            std::vector<uint8_t> out(S);
            lat[t].reserve(n_each);
            for (uint64_t i = 0; i < n_each; ++i) {
                const auto when = t0 + std::chrono::duration_cast<clk::duration>(
                                           std::chrono::duration<double>((i + double(t) / threads) / per_thread));
                std::this_thread::sleep_until(when);
                const uint32_t k = uint32_t((uint64_t(t) * 7919 + i) % pool);
                const int rc = mode == 0
                                   ? xpir_batcher_answer(static_cast<xpir_batcher*>(target), qpool + k * nb, N,
                                                         seeds + size_t(k) * 32, out.data())
                                   : xpir_answer_batch(static_cast<xpir_store*>(target), qpool + k * nb, nb, N, 1,
                                                       seeds + size_t(k) * 32, out.data());
                if (rc) {
                    first_rc = rc;
                    return;
                }
                lat[t].push_back(std::chrono::duration<double, std::micro>(clk::now() - when).count());
            }
        });
    for (auto& th : ts) th.join();
    const double wall = std::chrono::duration<double>(clk::now() - t0).count();
    std::vector<double> all;
    for (auto& v : lat) all.insert(all.end(), v.begin(), v.end());
    if (all.empty()) return first_rc ? first_rc.load() : -1;
    std::sort(all.begin(), all.end());
    auto pct = [&](double p) { return all[std::min(all.size() - 1, size_t(p * all.size()))]; };
    out6[0] = double(all.size()) / wall;
    out6[1] = pct(0.5);
    out6[2] = pct(0.9);
    out6[3] = pct(0.99);
    out6[4] = all.back();
    out6[5] = double(all.size());
    return first_rc;
}
