// Drop-in replacement for the reference's src/pir.cpp
// (/root/reference/proj/src/pir.cpp): the same declarations from
// oblog/pir.hpp, with the server-side scan (answer, answer_batch — pir.cpp:29-52)
// and the answer mask (mask_answer — pir.cpp:65-69) executed by the B200 kernels
// behind include/xpir.h. Link this TU instead of pir.cpp.
//
// Client-side helpers (gen_queries, reconstruct, combine_masked, unmask) are not
// on the server hot path. This TU replaces pir.cpp wholesale, so it must define
// them too: they restate the reference client code (pir.cpp:7-27, 54-82) with
// the same exception strings, kept only for link completeness.
//
// Which device image answers a pir::Snapshot:
//  * a snapshot sealed by the ServerCore drop-in (server_b200.cpp) is
//    registered with its device ring image at seal time (b200_dropin.hpp) and
//    answered from it directly — no upload and no per-call hashing;
//  * any other snapshot (e.g. one built from Table::snapshot()) is uploaded to
//    HBM on first use and cached, keyed by (data pointer, size, geometry, epoch)
//    plus a fixed 4,096-word sample of its bytes (sealed snapshots are
//    immutable by contract, server.hpp:70-71 / SPEC.md:178; the sample guards
//    against a new snapshot allocated at a freed one's address).
//
// Single answers (pir::answer — what server::answer_share calls per client
// read, from node.cpp's session and link threads concurrently) go through one
// read batcher per snapshot geometry (xpir_batcher_*), so concurrent reads are
// coalesced into one device scan; a lone caller is scanned at once.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <list>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>

#include "b200_dropin.hpp"
#include "oblog/pir.hpp"
#include "xpir.h"

namespace oblog::b200 {

namespace {
struct TraceStat {
    uint64_t calls = 0;
    double total_us = 0, max_us = 0;
};
struct TraceTable {
    std::mutex mu;
    std::map<std::string, TraceStat> stats;
    ~TraceTable() {
        if (stats.empty()) return;
        std::fprintf(stderr, "drop-in trace: entry, calls, total ms, mean us, max us\n");
        for (const auto& [k, v] : stats)
            std::fprintf(stderr, "  %-28s %9llu %10.1f %9.1f %9.1f\n", k.c_str(), (unsigned long long)v.calls,
                         v.total_us * 1e-3, v.total_us / double(v.calls), v.max_us);
    }
};
TraceTable* trace_table() {
    static const bool on = [] {
        const char* e = std::getenv("XPIR_DROPIN_TRACE");
        return e && *e && *e != '0';
    }();
    if (!on) return nullptr;
    static TraceTable t;
    return &t;
}
}  // namespace

Trace::Trace(const char* n) : name(n), t0(std::chrono::steady_clock::now()) {}
Trace::~Trace() {
    TraceTable* t = trace_table();
    if (!t) return;
    const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    std::lock_guard<std::mutex> lk(t->mu);
    TraceStat& st = t->stats[name];
    st.calls += 1;
    st.total_us += us;
    if (us > st.max_us) st.max_us = us;
}

void check(int rc, const char* what) {
    if (rc == XPIR_OK) return;
    std::string msg = std::string(what) + ": " + xpir_last_error();
    if (rc == XPIR_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

}  // namespace oblog::b200

namespace {

using oblog::b200::check;

// ---- registered (ServerCore-sealed) snapshots -------------------------------
struct Registered {
    xpir_store* st;
    uint64_t epoch;
    uint32_t buckets, bucket_size;
};
std::mutex g_reg_mu;
std::unordered_map<const void*, Registered>& registry() {
    static auto* m = new std::unordered_map<const void*, Registered>;  // leaked on purpose
    return *m;
}

// ---- uploaded snapshots ------------------------------------------------------
uint64_t sample_fingerprint(const oblog::pir::Snapshot& s) {
    // FNV-1a over 4,096 8-byte words spread evenly over the image (all of them
    // for images up to 32 KiB), plus the length: constant cost per call
    const uint8_t* p = s.data.data();
    const size_t n = s.data.size();
    uint64_t h = 1469598103934665603ULL ^ n;
    auto mix = [&](uint64_t w) { h = (h ^ w) * 1099511628211ULL; };
    const size_t words = n / 8;
    const size_t step = words <= 4096 ? 1 : words / 4096;
    for (size_t i = 0; i < words; i += step) {
        uint64_t w;
        std::memcpy(&w, p + 8 * i, 8);
        mix(w);
    }
    for (size_t i = words * 8; i < n; ++i) mix(p[i]);
    return h;
}

struct Resident {
    const void* ptr = nullptr;
    size_t size = 0;
    uint32_t buckets = 0, bucket_size = 0;
    uint64_t epoch = 0, fp = 0;
    xpir_store* st = nullptr;
    Resident() = default;
    Resident(const Resident&) = delete;
    Resident& operator=(const Resident&) = delete;
    ~Resident() {
        if (st) xpir_store_destroy(st);
    }
};

class StoreCache {
public:
    std::shared_ptr<Resident> get(const oblog::pir::Snapshot& s) {
        if (s.data.size() != size_t(s.bucket_count) * s.bucket_size)
            throw std::invalid_argument("pir: snapshot has no host bytes and no registered device image");
        const uint64_t fp = sample_fingerprint(s);
        std::lock_guard<std::mutex> lk(mu_);
        for (auto it = lru_.begin(); it != lru_.end(); ++it) {
            const auto& r = **it;
            if (r.ptr == s.data.data() && r.size == s.data.size() && r.buckets == s.bucket_count &&
                r.bucket_size == s.bucket_size && r.epoch == s.epoch && r.fp == fp) {
                lru_.splice(lru_.begin(), lru_, it);
                return lru_.front();
            }
        }
        auto r = std::make_shared<Resident>();
        check(xpir_store_create(0, s.bucket_count, s.bucket_size, 0, s.bucket_count, &r->st), "pir: store_create");
        r->ptr = s.data.data();
        r->size = s.data.size();
        r->buckets = s.bucket_count;
        r->bucket_size = s.bucket_size;
        r->epoch = s.epoch;
        r->fp = fp;
        check(xpir_store_upload(r->st, s.data.data(), s.epoch), "pir: store_upload");
        lru_.push_front(r);
        while (lru_.size() > kMax) lru_.pop_back();
        return r;
    }

private:
    // at least Config::epoch_ring (16, config.hpp:44) snapshots stay resident
    static constexpr size_t kMax = 16;
    std::mutex mu_;
    std::list<std::shared_ptr<Resident>> lru_;
};

StoreCache& cache() {
    // Intentionally leaked: device stores must not be freed from a static
    // destructor that may run after the CUDA runtime has shut down.
    static StoreCache* c = new StoreCache;
    return *c;
}

// The device image that answers `snap`; `keep` holds an uploaded one alive for
// the duration of the call (a registered image is held by its snapshot's owner).
struct Target {
    xpir_store* st = nullptr;
    std::shared_ptr<Resident> keep;
};
Target resolve(const oblog::pir::Snapshot& snap) {
    if (xpir_store* st = oblog::b200::registered_store(snap)) return {st, nullptr};
    auto r = cache().get(snap);
    return {r->st, r};
}

// One read batcher per snapshot geometry (leaked on purpose, like the cache):
// up to 1024 reads per scan, sealed at once while the device is idle, else
// 200 us after a batch's first read.
xpir_batcher* batcher_for(uint32_t N, uint32_t S) {
    static std::mutex mu;
    static auto* m = new std::map<std::pair<uint32_t, uint32_t>, xpir_batcher*>;
    std::lock_guard<std::mutex> lk(mu);
    auto& b = (*m)[{N, S}];
    if (!b) check(xpir_batcher_create_geometry(0, N, S, 1024, 200, &b), "pir: batcher_create");
    return b;
}

oblog::bytes scan_one(const oblog::pir::Snapshot& snap, const oblog::pir::QueryVector& q, const uint8_t* seed) {
    oblog::bytes out(snap.bucket_size, 0);
    if (snap.bucket_count == 0 || snap.bucket_size == 0) return out;
    const Target t = resolve(snap);
    check(xpir_batcher_answer_on(batcher_for(snap.bucket_count, snap.bucket_size), t.st, q.data.data(),
                                 snap.bucket_count, seed, out.data()),
          seed ? "answer_share" : "answer");
    return out;
}

}  // namespace

namespace oblog::b200 {

void register_snapshot(const pir::Snapshot* snap, xpir_store* st) {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    registry()[snap] = Registered{st, snap->epoch, snap->bucket_count, snap->bucket_size};
}

void unregister_snapshot(const pir::Snapshot* snap) {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    registry().erase(snap);
}

xpir_store* registered_store(const pir::Snapshot& snap) {
    std::lock_guard<std::mutex> lk(g_reg_mu);
    auto it = registry().find(&snap);
    if (it == registry().end()) return nullptr;
    const Registered& r = it->second;
    if (r.epoch != snap.epoch || r.buckets != snap.bucket_count || r.bucket_size != snap.bucket_size) return nullptr;
    return r.st;
}

bytes answer_masked(const pir::Snapshot& snap, const pir::QueryVector& q, const crypto::Seed& seed) {
    Trace tr("pir.answer_masked");
    if (q.bit_count != snap.bucket_count) throw std::invalid_argument("answer: query length mismatch");
    return scan_one(snap, q, seed.data());
}

}  // namespace oblog::b200

namespace oblog::pir {

// pir.cpp:7-27 (client side): servers-1 uniform shares, the last one their XOR
// with the unit vector at beta; unused trailing bits of the uniform shares cleared.
std::vector<QueryVector> gen_queries(uint32_t beta, uint32_t bucket_count, uint32_t servers, Rng& rng) {
    if (bucket_count == 0) throw std::invalid_argument("gen_queries: no buckets");
    if (servers < 2) throw std::invalid_argument("gen_queries: need at least 2 servers");
    if (beta >= bucket_count) throw std::invalid_argument("gen_queries: target out of range");
    std::vector<QueryVector> qs(servers, QueryVector::zero(bucket_count));
    const size_t nbytes = qs.front().data.size();
    const uint32_t tail = bucket_count % 8;
    QueryVector& last = qs.back();
    last.set(beta);
    for (uint32_t s = 0; s + 1 < servers; ++s) {
        uint8_t* d = qs[s].data.data();
        rng.fill(d, nbytes);
        if (tail) d[nbytes - 1] &= uint8_t(0xffu >> (8 - tail));
        xor_into(last.data.data(), d, nbytes);
    }
    return qs;
}

std::vector<bytes> answer_batch(const Snapshot& snap, const std::vector<QueryVector>& qs) {
    b200::Trace tr("pir.answer_batch");
    for (const QueryVector& q : qs)
        if (q.bit_count != snap.bucket_count) throw std::invalid_argument("answer_batch: query length mismatch");
    std::vector<bytes> out(qs.size(), bytes(snap.bucket_size, 0));
    if (qs.empty() || snap.bucket_count == 0 || snap.bucket_size == 0) return out;
    const Target t = resolve(snap);
    const size_t nb = (snap.bucket_count + 7) / 8;
    bytes rows(qs.size() * nb), flat(qs.size() * size_t(snap.bucket_size));
    for (size_t r = 0; r < qs.size(); ++r) std::memcpy(rows.data() + r * nb, qs[r].data.data(), nb);
    check(xpir_answer_batch(t.st, rows.data(), nb, snap.bucket_count, uint32_t(qs.size()), nullptr, flat.data()),
          "answer_batch");
    for (size_t r = 0; r < qs.size(); ++r)
        std::memcpy(out[r].data(), flat.data() + r * snap.bucket_size, snap.bucket_size);
    return out;
}

bytes answer(const Snapshot& snap, const QueryVector& q) {
    b200::Trace tr("pir.answer");
    if (q.bit_count != snap.bucket_count) throw std::invalid_argument("answer: query length mismatch");
    return scan_one(snap, q, nullptr);
}

// pir.cpp:54-63 (client / leader side): XOR of equally long answers
bytes reconstruct(const std::vector<bytes>& answers) {
    if (answers.empty()) throw std::invalid_argument("reconstruct: no answers");
    bytes acc(answers.front());
    for (auto it = answers.begin() + 1; it != answers.end(); ++it) {
        if (it->size() != acc.size()) throw std::invalid_argument("reconstruct: answer length mismatch");
        xor_into(acc.data(), it->data(), acc.size());
    }
    return acc;
}

// pir.cpp:65-69 — server side: pad generated and applied on device
bytes mask_answer(byte_view answer, const crypto::Seed& seed) {
    bytes out(answer.size());
    if (!answer.empty())
        check(xpir_mask_answer(answer.data(), answer.size(), seed.data(), out.data()), "mask_answer");
    return out;
}

bytes combine_masked(const std::vector<bytes>& masked) { return reconstruct(masked); }

// pir.cpp:75-82 (client side): strip every server's pad
bytes unmask(byte_view combined, const std::vector<crypto::Seed>& seeds) {
    bytes acc(combined.begin(), combined.end());
    for (const crypto::Seed& s : seeds) {
        const bytes pad = crypto::prng_expand(s, acc.size());
        xor_into(acc.data(), pad.data(), acc.size());
    }
    return acc;
}

}  // namespace oblog::pir
