// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" wrappers around the UNMODIFIED reference implementation
// (/root/reference/proj/src, compiled where it lies by oracle/Makefile into
// oracle/_ref/libxpir_ref.so). Used by tests/ to pin the C restatement
// (oracle/xpir_oracle.c) and the CUDA path, by oracle/make_golden.py to write
// tests/golden/, and by bench.py's reference / cpu_baseline legs.
//
// Every wrapper calls the reference function named in its comment; nothing here
// re-implements reference logic.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "oblog/crypto.hpp"
#include "oblog/cuckoo.hpp"
#include "oblog/notify.hpp"
#include "oblog/pir.hpp"
#include "oblog/rng.hpp"

using namespace oblog;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return -1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -2;
    }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// crypto::prng_expand (crypto.cpp:35-45)
int ref_prng_expand(const uint8_t* seed32, uint8_t* out, uint64_t len) {
    return guarded([&] {
        crypto::Seed s;
        std::memcpy(s.data(), seed32, 32);
        if (len) crypto::prng_expand_into(s, out, len);
    });
}

// crypto::prf (crypto.cpp:17-33)
int ref_prf(const uint8_t* key16, uint64_t input, uint64_t modulus, uint64_t* out) {
    return guarded([&] {
        crypto::PrfKey k;
        std::memcpy(k.data(), key16, 16);
        *out = crypto::prf(k, input, modulus);
    });
}

// crypto::bloom_positions (crypto.cpp:146-166)
int ref_bloom_positions(const uint8_t* item, uint64_t len, uint32_t h, uint32_t m, uint32_t* out) {
    return guarded([&] {
        auto v = crypto::bloom_positions(byte_view(item, len), h, m);
        std::copy(v.begin(), v.end(), out);
    });
}

// notify::make_interest (notify.cpp:30-35)
int ref_make_interest(uint32_t m, uint32_t h, const uint8_t* id16, uint64_t seq, uint32_t* out) {
    return guarded([&] {
        LogId id;
        std::memcpy(id.data(), id16, 16);
        auto v = notify::make_interest(notify::BloomParams{m, h}, id, seq);
        std::copy(v.begin(), v.end(), out);
    });
}

uint32_t ref_bloom_hash_count(uint32_t m, uint64_t n) { return notify::bloom_hash_count(m, n); }

// crypto::digest (crypto.cpp:168-175) — BLAKE2b
int ref_digest(const uint8_t* data, uint64_t len, uint64_t outlen, uint8_t* out) {
    return guarded([&] {
        auto d = crypto::digest(byte_view(data, len), outlen);
        std::memcpy(out, d.data(), outlen);
    });
}

// DetRng (rng.hpp:41-55, rng.cpp:18-44)
void* ref_detrng_new(uint64_t seed) { return new DetRng(seed); }
void* ref_detrng_new_key(const uint8_t* key32) {
    std::array<uint8_t, 32> k;
    std::memcpy(k.data(), key32, 32);
    return new DetRng(k);
}
void ref_detrng_free(void* r) { delete static_cast<DetRng*>(r); }
void ref_detrng_fill(void* r, uint8_t* out, uint64_t n) { static_cast<DetRng*>(r)->fill(out, n); }
uint64_t ref_detrng_next_u64(void* r) { return static_cast<DetRng*>(r)->next_u64(); }
uint64_t ref_detrng_uniform(void* r, uint64_t bound) { return static_cast<DetRng*>(r)->uniform(bound); }

// pir::gen_queries (pir.cpp:7-27); out = servers * ceil(N/8) bytes
int ref_gen_queries(uint32_t beta, uint32_t buckets, uint32_t servers, void* rng, uint8_t* out) {
    return guarded([&] {
        auto qs = pir::gen_queries(beta, buckets, servers, *static_cast<DetRng*>(rng));
        size_t nb = (buckets + 7) / 8;
        for (size_t i = 0; i < qs.size(); ++i) std::memcpy(out + i * nb, qs[i].data.data(), nb);
    });
}

// pir::Snapshot (pir.hpp:32-41) built from caller bytes
void* ref_snapshot_new(const uint8_t* db, uint32_t buckets, uint32_t bucket_size) {
    auto* s = new pir::Snapshot;
    s->epoch = 1;
    s->bucket_count = buckets;
    s->bucket_size = bucket_size;
    s->data.assign(db, db + size_t(buckets) * bucket_size);
    return s;
}
// Same, filled from a DetRng fill call (the §8(d) store recipe) without a host copy.
void* ref_snapshot_new_detrng(void* rng, uint32_t buckets, uint32_t bucket_size) {
    auto* s = new pir::Snapshot;
    s->epoch = 1;
    s->bucket_count = buckets;
    s->bucket_size = bucket_size;
    s->data.resize(size_t(buckets) * bucket_size);
    static_cast<DetRng*>(rng)->fill(s->data.data(), s->data.size());
    return s;
}
void ref_snapshot_free(void* s) { delete static_cast<pir::Snapshot*>(s); }
const uint8_t* ref_snapshot_data(void* s) { return static_cast<pir::Snapshot*>(s)->data.data(); }

// pir::answer (pir.cpp:29-39). q_bits = query bit count (must equal buckets or it throws).
int ref_answer(void* snap, const uint8_t* q, uint32_t q_bits, uint8_t* out) {
    return guarded([&] {
        const auto& s = *static_cast<pir::Snapshot*>(snap);
        pir::QueryVector qv;
        qv.bit_count = q_bits;
        qv.data.assign(q, q + (q_bits + 7) / 8);
        auto a = pir::answer(s, qv);
        std::memcpy(out, a.data(), a.size());
    });
}

// pir::answer_batch (pir.cpp:41-52), run on `threads` host threads, each calling
// the reference answer_batch on a disjoint contiguous slice of the requests over
// the one shared immutable Snapshot (allowed by SPEC.md:178). Returns the wall
// seconds of the answer_batch calls only (query-vector construction excluded).
int ref_answer_batch(void* snap, const uint8_t* qbits, uint64_t q_stride, uint32_t batch,
                     uint8_t* out, uint32_t threads, double* seconds) {
    return guarded([&] {
        const auto& s = *static_cast<pir::Snapshot*>(snap);
        const size_t nb = (s.bucket_count + 7) / 8;
        uint32_t T = std::max(1u, std::min(threads, batch ? batch : 1u));
        std::vector<std::vector<pir::QueryVector>> slices(T);
        std::vector<uint32_t> lo(T + 1);
        for (uint32_t t = 0; t <= T; ++t) lo[t] = uint32_t(uint64_t(batch) * t / T);
        for (uint32_t t = 0; t < T; ++t)
            for (uint32_t r = lo[t]; r < lo[t + 1]; ++r) {
                pir::QueryVector q;
                q.bit_count = s.bucket_count;
                q.data.assign(qbits + r * q_stride, qbits + r * q_stride + nb);
                slices[t].push_back(std::move(q));
            }
        std::vector<std::vector<bytes>> res(T);
        std::vector<std::string> errs(T);
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (uint32_t t = 0; t < T; ++t)
            pool.emplace_back([&, t] {
                try {
                    res[t] = pir::answer_batch(s, slices[t]);
                } catch (const std::exception& e) {
                    errs[t] = e.what();
                }
            });
        for (auto& th : pool) th.join();
        auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        for (uint32_t t = 0; t < T; ++t)
            if (!errs[t].empty()) throw std::invalid_argument(errs[t]);
        for (uint32_t t = 0; t < T; ++t)
            for (uint32_t r = lo[t]; r < lo[t + 1]; ++r)
                std::memcpy(out + size_t(r) * s.bucket_size, res[t][r - lo[t]].data(),
                            s.bucket_size);
    });
}

// pir::mask_answer (pir.cpp:65-69)
int ref_mask_answer(const uint8_t* ans, uint64_t len, const uint8_t* seed32, uint8_t* out) {
    return guarded([&] {
        crypto::Seed sd;
        std::memcpy(sd.data(), seed32, 32);
        auto m = pir::mask_answer(byte_view(ans, len), sd);
        std::memcpy(out, m.data(), len);
    });
}

// cuckoo::Table (cuckoo.hpp:37-84, cuckoo.cpp)
void* ref_table_new(uint32_t buckets, uint32_t depth, uint64_t capacity, uint64_t item_size,
                    const uint8_t* seed32) {
    try {
        crypto::Seed sd;
        std::memcpy(sd.data(), seed32, 32);
        return new cuckoo::Table(buckets, depth, capacity, item_size, sd);
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void ref_table_free(void* t) { delete static_cast<cuckoo::Table*>(t); }

// Table::insert (cuckoo.cpp:56-126) for n items; report[4*i..] = stored, dropped,
// gc_evicted, displacements.
int ref_table_insert_batch(void* t, const uint32_t* beta1, const uint32_t* beta2,
                           const uint8_t* payload, uint64_t n, uint32_t* report) {
    return guarded([&] {
        auto& tab = *static_cast<cuckoo::Table*>(t);
        cuckoo::Item it;
        for (uint64_t i = 0; i < n; ++i) {
            it.beta1 = beta1[i];
            it.beta2 = beta2[i];
            it.data.assign(payload + i * tab.item_size(), payload + (i + 1) * tab.item_size());
            auto r = tab.insert(it);
            if (report) {
                report[4 * i + 0] = r.stored;
                report[4 * i + 1] = r.dropped;
                report[4 * i + 2] = r.gc_evicted;
                report[4 * i + 3] = r.displacements;
            }
        }
    });
}

// Table::snapshot (cuckoo.cpp:128-135) bytes
void ref_table_data(void* t, uint8_t* out) {
    auto snap = static_cast<cuckoo::Table*>(t)->snapshot();
    std::memcpy(out, snap.data.data(), snap.data.size());
}
// Table::state_digest (cuckoo.cpp:137-149)
void ref_table_state_digest(void* t, uint8_t* out32) {
    auto d = static_cast<cuckoo::Table*>(t)->state_digest();
    std::memcpy(out32, d.data(), 32);
}
void ref_table_counters(void* t, uint64_t* writes, uint64_t* live) {
    auto* tab = static_cast<cuckoo::Table*>(t);
    *writes = tab->writes_applied();
    *live = tab->live_count();
}
int ref_table_slot_used(void* t, uint32_t b, uint32_t s) {
    return static_cast<cuckoo::Table*>(t)->slot_used(b, s) ? 1 : 0;
}

// notify::Window (notify.hpp:57-88, notify.cpp:54-117)
void* ref_window_new(uint32_t m, uint32_t h, uint32_t w) {
    try {
        return new notify::Window(notify::BloomParams{m, h}, w);
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void ref_window_free(void* w) { delete static_cast<notify::Window*>(w); }
int ref_window_absorb(void* w, const uint32_t* pos, uint64_t n) {
    return guarded([&] { static_cast<notify::Window*>(w)->absorb(std::span<const uint32_t>(pos, n)); });
}
void ref_window_rotate(void* w) { static_cast<notify::Window*>(w)->rotate(); }
void ref_window_digest(void* w, uint8_t* out32) {
    auto d = static_cast<notify::Window*>(w)->digest();
    std::memcpy(out32, d.data(), 32);
}
uint64_t ref_window_size(void* w) { return static_cast<notify::Window*>(w)->size(); }
uint64_t ref_window_base(void* w) { return static_cast<notify::Window*>(w)->base(); }
void ref_window_delta_words(void* w, uint64_t i, uint64_t* out) {
    const auto& d = static_cast<notify::Window*>(w)->delta(i);
    std::memcpy(out, d.words.data(), d.words.size() * 8);
}

// notify::encode_delta / decode_delta (notify.cpp:139-180), Window::digest(count)
int64_t ref_encode_delta(uint32_t m, const uint64_t* words, uint8_t* out, uint64_t cap) {
    notify::DeltaFilter d = notify::DeltaFilter::empty(m);
    std::memcpy(d.words.data(), words, d.words.size() * 8);
    bytes enc = notify::encode_delta(d);
    if (out && enc.size() <= cap) std::memcpy(out, enc.data(), enc.size());
    return int64_t(enc.size());
}
// 1 ok (m, words filled when words_cap suffices), 0 nullopt
int ref_decode_delta(const uint8_t* buf, uint64_t len, uint32_t* m, uint64_t* words, uint64_t words_cap) {
    auto d = notify::decode_delta(byte_view(buf, len));
    if (!d) return 0;
    *m = d->m_bits;
    if (words && d->words.size() <= words_cap) std::memcpy(words, d->words.data(), d->words.size() * 8);
    return 1;
}
// notify::encode_positions: encoded length, or -1 when the reference throws
// (the field capacity is exceeded); out receives the cap-byte field
int64_t ref_encode_positions(const uint32_t* positions, uint64_t n, uint8_t* out, uint64_t cap) {
    try {
        bytes enc = notify::encode_positions(std::span<const uint32_t>(positions, n), cap);
        std::memcpy(out, enc.data(), enc.size());
        return int64_t(enc.size());
    } catch (const std::invalid_argument&) {
        return -1;
    }
}
// the same for n writes of h positions (a server decoding / a client encoding a
// round's writes), timed by bench_codec.py: ok[i] = 0 where the reference throws
void ref_encode_positions_batch(const uint32_t* positions, uint32_t h, uint64_t n, uint64_t cap, uint8_t* out,
                                uint8_t* ok) {
    for (uint64_t i = 0; i < n; ++i) ok[i] = ref_encode_positions(positions + i * h, h, out + i * cap, cap) >= 0;
}
// count[i] = number of positions (written to pos[i*cap ..]) or 0xffffffff for nullopt
void ref_decode_positions_batch(const uint8_t* fields, uint64_t cap, uint64_t n, uint32_t* pos, uint32_t* count) {
    for (uint64_t i = 0; i < n; ++i) {
        auto p = notify::decode_positions(byte_view(fields + i * cap, cap));
        if (!p) {
            count[i] = 0xffffffffu;
            continue;
        }
        count[i] = uint32_t(p->size());
        for (size_t k = 0; k < p->size() && k < cap; ++k) pos[i * cap + k] = (*p)[k];
    }
}
// notify::decode_positions: 1 ok (count, positions when they fit), 0 nullopt
int ref_decode_positions(const uint8_t* buf, uint64_t len, uint32_t* out, uint32_t max_out, uint32_t* count) {
    auto p = notify::decode_positions(byte_view(buf, len));
    if (!p) return 0;
    *count = uint32_t(p->size());
    for (size_t i = 0; i < p->size() && i < max_out; ++i) out[i] = (*p)[i];
    return 1;
}
void ref_window_digest_n(void* w, uint64_t count, uint8_t* out32) {
    auto d = static_cast<notify::Window*>(w)->digest(count);
    std::memcpy(out32, d.data(), 32);
}

}  // extern "C"
