// Test / measurement infrastructure (not product code): the reference's own
// production-path benchmarks, linked against either the B200 drop-in TUs
// (bench_read_b200: pir_b200.cpp, cuckoo_b200.cpp, server_b200.cpp) or the
// unmodified reference TUs (bench_read_ref). Same source, same inputs.
//
//   bench_read process  N[,N...] [iters]       harness::bench_process_read (harness.cpp:429-476)
//   bench_read concurrent N threads reads      node-style: `threads` host threads call
//                                              server::answer_share on one sealed snapshot
//   bench_read writes   capacity writes_per_seal epochs
//                                              ServerCore::apply_write x k + seal_epoch (server.cpp:58-81)
//   bench_read delivery                        acceptance.cpp criterion 5's first replay (replay.cpp:222):
//                                              a real-time 3-server cluster, 8 chat users, 500 messages
//
// Each prints one JSON object per measurement on stdout.
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "oblog/config.hpp"
#include "oblog/crypto.hpp"
#include "oblog/cuckoo.hpp"
#include "oblog/harness.hpp"
#include "oblog/logproto.hpp"
#include "oblog/pir.hpp"
#include "oblog/server.hpp"
#include "oblog/wire.hpp"

using namespace oblog;
using clk = std::chrono::steady_clock;

static double since_us(clk::time_point t0) {
    return std::chrono::duration<double, std::micro>(clk::now() - t0).count();
}

static std::vector<uint64_t> parse_list(const char* s) {
    std::vector<uint64_t> v;
    for (const char* p = s; *p;) {
        v.push_back(std::strtoull(p, nullptr, 10));
        while (*p && *p != ',') ++p;
        if (*p == ',') ++p;
    }
    return v;
}

static int process(int argc, char** argv) {
    auto ns = parse_list(argc > 2 ? argv[2] : "10000,100000");
    const int iters = argc > 3 ? std::atoi(argv[3]) : 20;
    for (uint64_t n : ns) {
        auto t0 = clk::now();
        auto pt = harness::bench_process_read(n, 4, 1024, iters);
        std::printf("{\"bench\": \"bench_process_read\", \"n\": %llu, \"buckets\": %u, \"table_bytes\": %llu, "
                    "\"iters\": %d, \"mean_us\": %.2f, \"setup_and_run_s\": %.2f}\n",
                    (unsigned long long)pt.n, pt.buckets, (unsigned long long)pt.table_bytes, pt.iters, pt.mean_us,
                    since_us(t0) * 1e-6);
        std::fflush(stdout);
    }
    return 0;
}

// The same table and blob recipe as bench_process_read, answered by `threads`
// concurrent callers (node.cpp:263-266 / 528-530 call answer_share from the
// session and link threads outside state_mu_).
static int concurrent(int argc, char** argv) {
    const uint64_t n = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 100000;
    const int threads = argc > 3 ? std::atoi(argv[3]) : 64;
    const int reads = argc > 4 ? std::atoi(argv[4]) : 16;
    const uint32_t d = 4, z = 1024;
    const uint32_t b = uint32_t(std::ceil(double(n) / (Config::kDesignLoad * double(d))));
    const size_t item = logproto::item_data_len(z);
    DetRng rng(n ^ 0xC0C0);
    crypto::Seed tseed;
    rng.fill(tseed.data(), tseed.size());
    cuckoo::Table table(b, d, n, item, tseed);
    for (uint64_t i = 0; i < n; ++i) {
        cuckoo::Item it;
        it.beta1 = uint32_t(rng.uniform(b));
        it.beta2 = uint32_t(rng.uniform(b));
        it.data = rng.gen(item);
        table.insert(it);
    }
    auto snap = std::make_shared<pir::Snapshot>(table.snapshot());
    auto keys = crypto::box_keygen(rng);
    std::vector<bytes> blobs(size_t(threads) * reads);
    for (auto& blob : blobs) {
        auto q = pir::QueryVector::zero(b);
        rng.fill(q.data.data(), q.data.size());
        if (b % 8) q.data.back() &= uint8_t((1u << (b % 8)) - 1);
        crypto::Seed mask;
        rng.fill(mask.data(), mask.size());
        blob = crypto::pk_seal(keys.pk, wire::encode_read_share(q, mask), rng);
    }
    {  // warm: the snapshot's upload / first batch
        DetRng r2(1);
        server::answer_share(*snap, keys, blobs[0], b, r2);
    }
    std::atomic<int> go{0};
    std::atomic<uint64_t> bad{0};
    std::vector<std::thread> th;
    for (int t = 0; t < threads; ++t)
        th.emplace_back([&, t] {
            DetRng r(uint64_t(t) + 77);
            while (!go.load()) std::this_thread::yield();
            for (int k = 0; k < reads; ++k) {
                auto ans = server::answer_share(*snap, keys, blobs[size_t(t) * reads + k], b, r);
                if (ans.block.size() != size_t(d) * item) bad += 1;
            }
        });
    auto t0 = clk::now();
    go = 1;
    for (auto& x : th) x.join();
    const double us = since_us(t0);
    std::printf("{\"bench\": \"concurrent_answer_share\", \"n\": %llu, \"buckets\": %u, \"table_bytes\": %llu, "
                "\"threads\": %d, \"reads\": %d, \"wall_ms\": %.2f, \"reads_per_s\": %.1f, \"bad\": %llu}\n",
                (unsigned long long)n, b, (unsigned long long)snap->data.size(), threads, threads * reads, us * 1e-3,
                threads * reads / (us * 1e-6), (unsigned long long)bad.load());
    return 0;
}

// ServerCore write path: `epochs` x (writes_per_seal apply_write + seal_epoch).
static int writes(int argc, char** argv) {
    const uint64_t capacity = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 131072;
    const uint64_t per_seal = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 500;
    const int epochs = argc > 4 ? std::atoi(argv[4]) : 8;
    DetRng rng(4242);
    Config cfg = make_local_config(2, rng);
    cfg.capacity_n = capacity;
    cfg.depth_d = 4;
    cfg.message_z = 976;  // item = z + 48 = 1,024-byte slots
    cfg.epoch_ring = 16;
    server::ServerCore core(cfg, 0);
    const uint32_t buckets = cfg.buckets();
    auto bp = cfg.bloom_params();
    std::vector<logproto::WriteRequest> ws(per_seal * epochs);
    for (auto& w : ws) w = logproto::fake_write(buckets, cfg.message_z, bp, rng);
    double apply_us = 0, seal_us = 0;
    for (int e = 0; e < epochs; ++e) {
        auto t0 = clk::now();
        for (uint64_t i = 0; i < per_seal; ++i) core.apply_write(ws[e * per_seal + i], false);
        apply_us += since_us(t0);
        t0 = clk::now();
        core.seal_epoch();
        seal_us += since_us(t0);
    }
    std::printf("{\"bench\": \"servercore_writes\", \"capacity\": %llu, \"buckets\": %u, \"table_bytes\": %llu, "
                "\"writes_per_seal\": %llu, \"epochs\": %d, \"apply_write_us\": %.2f, \"seal_epoch_ms\": %.3f, "
                "\"epoch_ms\": %.3f, \"writes_per_s\": %.1f, \"latest_epoch\": %llu}\n",
                (unsigned long long)capacity, buckets, (unsigned long long)(uint64_t(buckets) * 4 * 1024),
                (unsigned long long)per_seal, epochs, apply_us / double(per_seal * epochs), seal_us * 1e-3 / epochs,
                (apply_us + seal_us) * 1e-3 / epochs, double(per_seal * epochs) / ((apply_us + seal_us) * 1e-6),
                (unsigned long long)core.latest_epoch());
    return 0;
}

// The cluster and chat workload of acceptance criterion 5 (acceptance.cpp:247-290,
// delivery_config), timed alone: wall-clock delivery latency through the nodes.
static int delivery(int, char**) {
    DetRng rng(555);
    Config cfg = make_local_config(3, rng);
    cfg.capacity_n = 4096;
    cfg.depth_d = 4;
    cfg.message_z = 256;
    cfg.write_interval_ms = 200;
    cfg.read_interval_ms = 100;
    cfg.jitter_ms = 0;
    cfg.get_updates_every = 2;
    cfg.giv_rotate_writes = 16;
    cfg.window_deltas = 100;
    cfg.epoch_seal_writes = 64;
    cfg.epoch_seal_interval_ms = 50;
    cfg.rate_limit = false;
    harness::ChatGenSpec spec;
    spec.users = 8;
    spec.channels = 1;
    spec.messages = 500;
    spec.interval_ms = 300;
    spec.seed = 11;
    auto msgs = harness::generate_chat(spec);
    auto t0 = clk::now();
    auto rep = harness::replay_workload(msgs, cfg, 7, 30000);
    std::printf("{\"bench\": \"delivery\", \"delivered\": %zu, \"expected\": %zu, \"latency_mean_ms\": %.1f, "
                "\"latency_p50_ms\": %.1f, \"latency_p95_ms\": %.1f, \"latency_max_ms\": %.1f, "
                "\"server_reads_per_s\": %.1f, \"wall_s\": %.1f}\n",
                rep.deliveries, rep.expected_deliveries, rep.latency_mean_ms, rep.latency_p50_ms,
                rep.latency_p95_ms, rep.latency_max_ms, rep.server_reads_per_sec, since_us(t0) * 1e-6);
    return 0;
}

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "process";
    if (mode == "process") return process(argc, argv);
    if (mode == "concurrent") return concurrent(argc, argv);
    if (mode == "writes") return writes(argc, argv);
    if (mode == "delivery") return delivery(argc, argv);
    std::fprintf(stderr, "usage: bench_read process|concurrent|writes|delivery ...\n");
    return 2;
}
