// Drop-in replacement for the reference's src/cuckoo.cpp
// (/root/reference/proj/src/cuckoo.cpp): oblog::cuckoo::Table with its state
// held in HBM and every mutation executed by the B200 write-path kernels
// (k_cuckoo_walk + payload gather/scatter) behind include/xpir.h.
//
// The class layout in oblog/cuckoo.hpp is unchanged. The device handle is kept
// in the payload member data_ (8 bytes; the payloads themselves live in HBM), so
// it follows the Table through moves (e.g. a growing std::vector<Table>); a
// copied Table shares its device state. The header's inline accessors
// (writes_applied, live_count, buckets, depth, item_size) read the scalar
// members, which insert() refreshes from the device counters. The reference
// header declares no destructor, so a device table lives until process exit;
// INTEGRATION.md shows the one-line header change (a pimpl member) a
// maintainer would make instead.
#include <cstring>
#include <stdexcept>
#include <string>

#include "oblog/cuckoo.hpp"
#include "xpir.h"

namespace {

void xpir_check(int rc, const char* what) {
    if (rc == XPIR_OK) return;
    std::string msg = std::string(what) + ": " + xpir_last_error();
    if (rc == XPIR_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

xpir_table* dev(const oblog::bytes& anchor) {
    if (anchor.size() != sizeof(xpir_table*)) throw std::logic_error("cuckoo: table has no device state (moved from?)");
    xpir_table* t = nullptr;
    std::memcpy(&t, anchor.data(), sizeof t);
    return t;
}

}  // namespace

namespace oblog::cuckoo {

Table::Table(uint32_t buckets, uint32_t depth, uint64_t capacity, size_t item_size,
             const crypto::Seed& seed)
    : buckets_(buckets), depth_(depth), capacity_(capacity), item_size_(item_size), rng_(seed) {
    // cuckoo.cpp:15-18
    if (buckets == 0 || depth == 0 || item_size == 0)
        throw std::invalid_argument("cuckoo: table dimensions must be positive");
    if (capacity == 0 || capacity > uint64_t(buckets) * depth)
        throw std::invalid_argument("cuckoo: capacity must be in [1, buckets*depth]");
    xpir_table* t = nullptr;
    xpir_check(xpir_table_create(0, buckets, depth, capacity, item_size, seed.data(), &t), "cuckoo: create");
    data_.resize(sizeof t);
    std::memcpy(data_.data(), &t, sizeof t);
}

InsertReport Table::insert(const Item& item) {
    // cuckoo.cpp:57-60
    if (item.beta1 >= buckets_ || item.beta2 >= buckets_)
        throw std::invalid_argument("cuckoo: bucket index out of range");
    if (item.data.size() != item_size_) throw std::invalid_argument("cuckoo: item size mismatch");
    xpir_table* t = dev(data_);
    uint32_t rep[4] = {0, 0, 0, 0};
    xpir_check(xpir_table_insert_batch(t, &item.beta1, &item.beta2, item.data.data(), 1, rep), "cuckoo: insert");
    xpir_check(xpir_table_counters(t, &writes_applied_, &live_, &next_stamp_), "cuckoo: counters");
    InsertReport r;
    r.stored = rep[0] != 0;
    r.dropped = rep[1] != 0;
    r.gc_evicted = rep[2] != 0;
    r.displacements = rep[3];
    return r;
}

pir::Snapshot Table::snapshot() const {  // cuckoo.cpp:128-135
    pir::Snapshot snap;
    snap.epoch = writes_applied_;
    snap.bucket_count = buckets_;
    snap.bucket_size = depth_ * uint32_t(item_size_);
    snap.data.resize(size_t(buckets_) * depth_ * item_size_);
    xpir_check(xpir_table_snapshot(dev(data_), snap.data.data()), "cuckoo: snapshot");
    return snap;
}

bytes Table::state_digest() const {  // cuckoo.cpp:137-149
    bytes out(32);
    xpir_check(xpir_table_state_digest(dev(data_), out.data()), "cuckoo: state_digest");
    return out;
}

std::optional<Table::Loc> Table::locate(byte_view data) const {  // cuckoo.cpp:151-158 (test helper)
    if (data.size() != item_size_) return std::nullopt;
    const size_t slots = size_t(buckets_) * depth_;
    bytes img(slots * item_size_), used(slots);
    xpir_check(xpir_table_snapshot(dev(data_), img.data()), "cuckoo: locate");
    xpir_check(xpir_table_meta(dev(data_), used.data(), nullptr, nullptr, nullptr), "cuckoo: locate");
    for (uint32_t b = 0; b < buckets_; ++b)
        for (uint32_t s = 0; s < depth_; ++s) {
            const size_t f = size_t(b) * depth_ + s;
            if (used[f] && std::memcmp(img.data() + f * item_size_, data.data(), item_size_) == 0)
                return Loc{b, s};
        }
    return std::nullopt;
}

bool Table::slot_used(uint32_t bucket, uint32_t slot) const {  // cuckoo.cpp:160-163
    const int rc = xpir_table_slot_used(dev(data_), bucket, slot);
    if (rc < 0) xpir_check(rc, "cuckoo: slot_used");
    return rc == 1;
}

}  // namespace oblog::cuckoo
