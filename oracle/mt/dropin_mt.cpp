// Test infrastructure (not product code): node.cpp-style concurrency on the
// drop-in pir TU. 64 host threads call pir::answer + pir::mask_answer — the
// scan + mask of server::answer_share (server.cpp:122-123) — against one sealed
// Snapshot at once, as the session and link threads do (node.cpp:263-266,
// 528-530). Linked against paper_2001_08250_b200/cpp/pir_b200.cpp, so the
// answers go through the read batcher. The checker is a plain host XOR of the
// selected buckets (pir.cpp:29-39) and the reference's own prng_expand
// (crypto.cpp:35-45, libsodium) for the pad.
#include <atomic>
#include <cstdio>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include "oblog/crypto.hpp"
#include "oblog/pir.hpp"

using namespace oblog;

int main() {
    const uint32_t N = 2000, S = 1024, T = 64, R = 12;
    std::mt19937_64 g(2001);
    pir::Snapshot snap;
    snap.bucket_count = N;
    snap.bucket_size = S;
    snap.epoch = 7;
    snap.data.resize(size_t(N) * S);
    for (auto& b : snap.data) b = uint8_t(g());
    std::vector<pir::QueryVector> qs;
    std::vector<crypto::Seed> seeds(T * R);
    for (uint32_t k = 0; k < T * R; ++k) {
        pir::QueryVector q = pir::QueryVector::zero(N);
        for (uint32_t j = 0; j < N; ++j)
            if (g() & 1) q.set(j);
        qs.push_back(q);
        for (auto& x : seeds[k]) x = uint8_t(g());
    }
    std::vector<bytes> got(T * R);
    std::vector<std::thread> ts;
    for (uint32_t t = 0; t < T; ++t)
        ts.emplace_back([&, t] {
            for (uint32_t r = 0; r < R; ++r) {
                const uint32_t k = t * R + r;
                bytes ans = pir::answer(snap, qs[k]);
                got[k] = pir::mask_answer(ans, seeds[k]);
            }
        });
    for (auto& th : ts) th.join();
    uint32_t bad = 0;
    for (uint32_t k = 0; k < T * R; ++k) {
        bytes want(S, 0);
        for (uint32_t j = 0; j < N; ++j)
            if (qs[k].data[j / 8] >> (j % 8) & 1)
                for (uint32_t b = 0; b < S; ++b) want[b] ^= snap.data[size_t(j) * S + b];
        bytes pad = crypto::prng_expand(seeds[k], S);
        for (uint32_t b = 0; b < S; ++b) want[b] ^= pad[b];
        if (got[k] != want) ++bad;
    }
    std::printf("dropin_mt: %u threads x %u reads, %u mismatches\n", T, R, bad);
    return bad ? 1 : 0;
}
