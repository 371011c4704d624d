// Drop-in replacement for the reference's src/server.cpp
// (/root/reference/proj/src/server.cpp): oblog::server::ServerCore and
// answer_share with the replica state held in HBM and driven by the device
// state machine behind include/xpir.h (xpir_server_*: cuckoo table + interest
// window + ring of sealed images).
//
//  * apply_write (server.cpp:58-73) = one xpir_server_apply_round of one write:
//    insert (device walk + payload scatter), absorb, rotate on the cadence.
//  * seal_epoch (server.cpp:75-81) seals on device: the ring's oldest image is
//    re-sealed in place from the slots rewritten since (no full-table copy, no
//    host copy). The pir::Snapshot handed out for the epoch carries epoch and
//    geometry and is registered with its device image (b200_dropin.hpp), which
//    stays pinned while any shared_ptr to the snapshot lives — the reference's
//    shared_ptr lifetime rule (server.cpp:83-87), kept on device.
//  * answer_share (server.cpp:115-135): pk_open and decode_read_share stay on the
//    host (the reference's own crypto.cpp / wire.cpp); scan + mask are ONE device
//    trip through the read batcher, coalesced with concurrent readers.
//
// Host bytes of sealed snapshots: the reference fills Snapshot::data with a full
// copy of the table at every seal. Here `data` stays empty unless the process
// sets OBLOG_B200_HOST_SNAPSHOTS=1 (then the device image is also copied out at
// seal time). Every reference caller of a sealed snapshot goes through
// pir::answer / answer_share / state_digest, which use the device image; code
// that reads snap->data directly needs the variable.
//
// The class layout of oblog/server.hpp is unchanged: the device state rides in
// epochs_ under a sentinel key (UINT64_MAX, never a real epoch; hidden from every
// accessor), so it follows the object through moves and is released with it
// (kept alive until the last snapshot of it is released). The members table_ /
// window_ are constructed only for the reference's argument checks; the state
// lives on device.
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>

#include "b200_dropin.hpp"
#include "oblog/server.hpp"
#include "xpir.h"

namespace oblog::server {
namespace {

using b200::check;

constexpr uint64_t kSentinel = std::numeric_limits<uint64_t>::max();

struct CoreState {
    xpir_server* sv = nullptr;
    xpir_table* table = nullptr;
    xpir_window* window = nullptr;
    uint32_t buckets = 0, bucket_size = 0;
    size_t item = 0;
    // encoded frozen deltas by absolute delta number (Window::base() + index): a
    // frozen delta never changes again, so each is encoded once, not at every freeze
    std::mutex enc_mu;
    std::map<uint64_t, bytes> enc_cache;
    CoreState() = default;
    CoreState(const CoreState&) = delete;
    CoreState& operator=(const CoreState&) = delete;
    ~CoreState() {
        if (sv) xpir_server_destroy(sv);
    }
};

// The device state rides in epochs_ under the sentinel key as an Anchor
// snapshot, so it follows the ServerCore through moves and copies (e.g. a
// std::vector<ServerCore> growing) and dies with the last of them.
struct Anchor : pir::Snapshot {
    std::shared_ptr<CoreState> cs;
};

template <class Map>
std::shared_ptr<CoreState> state_in(const Map& epochs) {
    auto it = epochs.find(kSentinel);
    if (it == epochs.end()) throw std::logic_error("server: ServerCore has no device state (moved from?)");
    return static_cast<const Anchor*>(it->second.get())->cs;
}

bool host_snapshots() {
    static const bool on = [] {
        const char* e = std::getenv("OBLOG_B200_HOST_SNAPSHOTS");
        return e && e[0] == '1';
    }();
    return on;
}

// The pir::Snapshot object for a sealed epoch: registered with its pinned device
// image; the deleter unregisters, unpins and frees it.
std::shared_ptr<const pir::Snapshot> sealed_snapshot(const std::shared_ptr<CoreState>& cs, uint64_t epoch) {
    xpir_store* st = nullptr;
    check(xpir_server_snapshot_acquire(cs->sv, epoch, &st, nullptr), "server: snapshot");
    auto* snap = new pir::Snapshot;
    snap->epoch = epoch;
    snap->bucket_count = cs->buckets;
    snap->bucket_size = cs->bucket_size;
    if (host_snapshots()) {
        snap->data.resize(size_t(cs->buckets) * cs->bucket_size);
        const int rc = xpir_store_download(st, 0, snap->data.size(), snap->data.data());
        if (rc) {
            xpir_server_snapshot_release(cs->sv, st);
            delete snap;
            check(rc, "server: snapshot host copy");
        }
    }
    b200::register_snapshot(snap, st);
    return std::shared_ptr<const pir::Snapshot>(snap, [cs, st](const pir::Snapshot* p) {
        b200::unregister_snapshot(p);
        xpir_server_snapshot_release(cs->sv, st);
        delete p;
    });
}

// cuckoo.cpp:15-18: the table dimension checks the reference's table_ member
// runs before anything else in the constructor; the member itself is a 1-slot
// placeholder (the real table is the device server's).
uint32_t checked_dims(const Config& cfg) {
    const uint32_t b = cfg.buckets();
    if (b == 0 || cfg.depth_d == 0 || cfg.item_size() == 0)
        throw std::invalid_argument("cuckoo: table dimensions must be positive");
    if (cfg.capacity_n == 0 || cfg.capacity_n > uint64_t(b) * cfg.depth_d)
        throw std::invalid_argument("cuckoo: capacity must be in [1, buckets*depth]");
    return 1;
}

bytes freeze_message(const WindowFreeze& f) {  // "window-sig-v1" || BE64 base || BE64 newest || digest
    bytes m = to_bytes("window-sig-v1");
    append_u64be(m, f.base);
    append_u64be(m, f.newest);
    append_bytes(m, f.digest);
    return m;
}

}  // namespace

crypto::Signature sign_freeze(const crypto::SecretKey& sign_seed, const WindowFreeze& f) {
    return crypto::sign(sign_seed, freeze_message(f));
}

bool verify_freeze(const crypto::PublicKey& pk, const WindowFreeze& f, const crypto::Signature& sig) {
    return crypto::verify(pk, freeze_message(f), sig);
}

ServerCore::ServerCore(const Config& cfg, uint32_t index)
    : cfg_(cfg),
      index_(index),
      table_(checked_dims(cfg), 1, 1, 1, cfg.s_cuckoo),
      window_(cfg.bloom_params(), cfg.window_deltas) {
    cfg_.validate();
    if (index >= cfg_.servers.size()) throw std::invalid_argument("server index out of range");
    const auto& me = cfg_.servers[index];
    if (!me.box_sk || !me.sign_sk)
        throw std::invalid_argument("server config is missing this server's secret keys");
    box_keys_ = crypto::BoxKeyPair{me.box_pk, *me.box_sk};
    sign_seed_ = *me.sign_sk;

    // the device replica: creation rotates the window once and seals epoch 1
    // (server.cpp:40-42)
    auto cs = std::make_shared<CoreState>();
    cs->buckets = cfg_.buckets();
    cs->item = cfg_.item_size();
    cs->bucket_size = uint32_t(cfg_.depth_d * cs->item);
    const notify::BloomParams bp = cfg_.bloom_params();
    check(xpir_server_create(0, cs->buckets, cfg_.depth_d, cfg_.capacity_n, cs->item, cfg_.s_cuckoo.data(),
                             bp.m_bits, bp.h, cfg_.window_deltas, cfg_.rotate_writes(), cfg_.epoch_ring, &cs->sv),
          "server: create");
    // start-up reservation: every ring image and the per-write scratch allocated now,
    // so no apply_write / seal_epoch allocates device memory
    check(xpir_server_reserve(cs->sv, 64), "server: reserve");
    check(xpir_server_info(cs->sv, nullptr, &latest_epoch_, nullptr, &cs->table, &cs->window), "server: info");
    auto anchor = std::make_shared<Anchor>();
    anchor->cs = cs;
    epochs_[kSentinel] = anchor;
    freeze_ = make_freeze();
    epochs_[latest_epoch_] = sealed_snapshot(cs, latest_epoch_);
}

WindowFreeze ServerCore::make_freeze() const {  // server.cpp:45-56, from the device window
    b200::Trace tr("server.make_freeze");
    auto cs = state_in(epochs_);
    WindowFreeze f;
    uint64_t count = 0;
    f.digest.resize(32);
    check(xpir_server_freeze(cs->sv, &f.base, &f.newest, f.digest.data(), &count), "server: freeze");
    // deltas 0..count-1 are frozen (server.cpp:46-48); the reference re-encodes all
    // of them every freeze, here only the ones not encoded before (one per rotation)
    std::lock_guard<std::mutex> lk(cs->enc_mu);
    cs->enc_cache.erase(cs->enc_cache.begin(), cs->enc_cache.lower_bound(f.base));
    for (uint64_t k = 0; k < count; ++k) {
        auto it = cs->enc_cache.find(f.base + k);
        if (it == cs->enc_cache.end()) {
            uint64_t len = 0;
            check(xpir_window_encode_delta(cs->window, k, nullptr, 0, &len), "server: encode_delta");
            bytes enc(len);
            check(xpir_window_encode_delta(cs->window, k, enc.data(), len, &len), "server: encode_delta");
            it = cs->enc_cache.emplace(f.base + k, std::move(enc)).first;
        }
        f.deltas.push_back(it->second);
    }
    return f;
}

ServerCore::ApplyResult ServerCore::apply_write(const logproto::WriteRequest& w, bool seal_after) {
    b200::Trace tr("server.apply_write");
    auto cs = state_in(epochs_);
    // server.cpp:60-61, then Table::insert's own size check (cuckoo.cpp:59-60)
    if (w.beta1 >= cs->buckets || w.beta2 >= cs->buckets)
        throw std::invalid_argument("write targets a bucket outside the table");
    if (w.data.size() != cs->item) throw std::invalid_argument("cuckoo: item size mismatch");
    ApplyResult out;
    uint32_t rep[4] = {0, 0, 0, 0};
    // insert, absorb, and the rotation on the cadence (server.cpp:63-70); an
    // out-of-range interest position throws after the insert, as the reference
    // (notify.cpp:62) — writes_applied does not advance then
    check(xpir_server_apply_round(cs->sv, &w.beta1, &w.beta2, w.data.data(), w.interest.data(),
                                  uint32_t(w.interest.size()), 1, 0, rep, nullptr),
          "server: apply_write");
    out.insert.stored = rep[0] != 0;
    out.insert.dropped = rep[1] != 0;
    out.insert.gc_evicted = rep[2] != 0;
    out.insert.displacements = rep[3];
    ++writes_applied_;
    if (writes_applied_ % cfg_.rotate_writes() == 0) {
        freeze_ = make_freeze();
        out.freeze = freeze_;
    }
    if (seal_after) out.sealed_epoch = seal_epoch();
    return out;
}

uint64_t ServerCore::seal_epoch() {
    b200::Trace tr("server.seal_epoch");
    auto cs = state_in(epochs_);
    // The epoch that falls off the ring (server.cpp:79) is released before the
    // device seal, so its image is re-sealed in place unless a reader still holds it.
    size_t real = epochs_.size() - epochs_.count(kSentinel);
    while (real >= cfg_.epoch_ring && real > 0) {
        epochs_.erase(epochs_.begin());
        --real;
    }
    uint64_t e = 0;
    check(xpir_server_seal(cs->sv, &e), "server: seal_epoch");
    latest_epoch_ = e;
    epochs_[e] = sealed_snapshot(cs, e);
    return latest_epoch_;
}

std::shared_ptr<const pir::Snapshot> ServerCore::snapshot_at(uint64_t epoch) const {
    b200::Trace tr("server.snapshot_at");
    if (epoch == kSentinel) return nullptr;
    auto it = epochs_.find(epoch);
    if (it == epochs_.end()) return nullptr;
    return it->second;
}

std::shared_ptr<const pir::Snapshot> ServerCore::latest_snapshot() const { return snapshot_at(latest_epoch_); }

crypto::Signature ServerCore::sign_current_freeze() const {
    b200::Trace tr("server.sign_current_freeze");
    return sign_freeze(sign_seed_, freeze_);
}

// server.cpp:95-113: every field the replicas must agree on; the table, the
// window and each sealed epoch's bytes are digested from the device state.
bytes ServerCore::state_digest() const {
    b200::Trace tr("server.state_digest");
    auto cs = state_in(epochs_);
    crypto::Hasher h(32);
    h.update(to_bytes("server-state-v1"));
    h.update_u64(writes_applied_);
    h.update_u64(latest_epoch_);
    bytes td(32), wd(32);
    check(xpir_table_state_digest(cs->table, td.data()), "server: table digest");
    check(xpir_window_digest(cs->window, wd.data()), "server: window digest");
    h.update(td);
    h.update(wd);
    h.update_u64(freeze_.base);
    h.update_u64(freeze_.newest);
    h.update(freeze_.digest);
    h.update_u64(epochs_.size() - epochs_.count(kSentinel));
    const size_t chunk = size_t(64) << 20;
    bytes buf;
    for (const auto& [num, snap] : epochs_) {
        if (num == kSentinel) continue;
        h.update_u64(num);
        xpir_store* st = b200::registered_store(*snap);
        if (!st) throw std::logic_error("server: sealed snapshot lost its device image");
        const size_t n = size_t(snap->bucket_count) * snap->bucket_size;
        crypto::Hasher d(32);  // crypto::digest(snap->data), streamed from HBM
        for (size_t off = 0; off < n; off += chunk) {
            const size_t len = std::min(chunk, n - off);
            buf.resize(len);
            check(xpir_store_download(st, off, len, buf.data()), "server: snapshot digest");
            d.update(buf);
        }
        h.update(d.finish());
    }
    return h.finish();
}

// server.cpp:115-135. Unsealing and parsing the share stay on the host; a bad
// blob earns a random block from the caller's rng, never an error.
ShareAnswer answer_share(const pir::Snapshot& snap, const crypto::BoxKeyPair& keys, byte_view blob,
                         uint32_t buckets, Rng& rng, ServerMetrics* metrics) {
    b200::Trace tr("server.answer_share");
    ShareAnswer out;
    if (auto plain = crypto::pk_open(keys, blob)) {
        auto share = wire::decode_read_share(*plain, buckets);
        if (share && share->first.bit_count == snap.bucket_count) {
            out.block = b200::answer_masked(snap, share->first, share->second);
            if (metrics) metrics->reads_answered += 1;
            return out;
        }
    }
    if (metrics) {
        metrics->decrypt_failures += 1;
        metrics->reads_answered += 1;
    }
    out.block = rng.gen(snap.bucket_size);
    return out;
}

}  // namespace oblog::server
