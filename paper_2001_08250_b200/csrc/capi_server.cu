// C-ABI (include/xpir.h): the device ServerCore — server::ServerCore (server.cpp:28-91).
#include "capi_internal.cuh"

// ===========================================================================
// replica state machine — server::ServerCore (server.hpp:57-98, server.cpp:28-91)
// on device: cuckoo table + interest window + a ring of sealed stores.
// ===========================================================================

static int server_seal(xpir_server* sv, uint64_t* epoch_out) {  // server.cpp:75-81
    xpir_table* t = sv->table;
    DeviceGuard g(sv->device);
    xpir_server::Sealed e{};
    bool incremental = false;
    if (sv->ring.size() >= sv->epoch_ring) {
        // the oldest epoch leaves the ring (server.cpp:79); its image is reused
        // unless a reader still holds it, in which case it is retired until released
        e = sv->ring.front();
        sv->ring.pop_front();
        if (e.pins) {
            sv->retired.push_back(e);
            e = xpir_server::Sealed{};
        } else {
            incremental = true;
        }
    }
    if (incremental) {
        // only slots rewritten since this image was sealed are copied
        XCK(launch_seal_incremental(t->d, t->lo, t->hi, e.since_batch, t->data, e.st->data, num_sms(sv->device),
                                    t->stream));
        count_launches(1);
    } else {
        if (!sv->spare.empty()) {
            e.st = sv->spare.back();
            sv->spare.pop_back();
        } else {
            int rc = xpir_store_create(sv->device, t->d.buckets, uint32_t(t->d.depth * t->d.item), t->lo, t->hi,
                                       &e.st);
            if (rc) return rc;
        }
        XCK(cudaMemcpyAsync(e.st->data, t->data, e.st->bytes(), cudaMemcpyDeviceToDevice, t->stream));
    }
    XCK(cudaStreamSynchronize(t->stream));
    e.pins = 0;
    e.since_batch = t->h.batch_id;
    e.epoch = ++sv->latest_epoch;
    e.st->epoch = e.epoch;
    sv->ring.push_back(e);
    if (epoch_out) *epoch_out = e.epoch;
    return XPIR_OK;
}

extern "C" {

int xpir_server_create(int device, uint32_t buckets, uint32_t depth, uint64_t capacity, uint64_t item_size,
                       const uint8_t seed[32], uint32_t m_bits, uint32_t h, uint32_t window_deltas,
                       uint32_t rotate_writes, uint32_t epoch_ring, xpir_server** out) {
    return xpir_server_create_shard(device, buckets, depth, capacity, item_size, seed, m_bits, h, window_deltas,
                                    rotate_writes, epoch_ring, 0, buckets, out);
}

int xpir_server_create_shard(int device, uint32_t buckets, uint32_t depth, uint64_t capacity, uint64_t item_size,
                             const uint8_t seed[32], uint32_t m_bits, uint32_t h, uint32_t window_deltas,
                             uint32_t rotate_writes, uint32_t epoch_ring, uint32_t lo, uint32_t hi,
                             xpir_server** out) {
    if (!out) return fail(XPIR_EINVAL, "server_create: null out");
    if (rotate_writes == 0) return fail(XPIR_EINVAL, "server_create: rotate_writes must be positive");
    if (epoch_ring == 0) return fail(XPIR_EINVAL, "server_create: epoch_ring must be positive");
    auto* sv = new xpir_server;
    sv->device = device;
    sv->rotate_writes = rotate_writes;
    sv->epoch_ring = epoch_ring;
    int rc = xpir_table_create_shard(device, buckets, depth, capacity, item_size, seed, lo, hi, &sv->table);
    if (!rc) rc = xpir_window_create(device, m_bits, h, window_deltas, &sv->window);
    if (!rc) rc = xpir_window_rotate(sv->window);  // server.cpp:40
    if (!rc) rc = server_seal(sv, nullptr);          // server.cpp:42, epoch 1 (all zeros)
    if (rc) {
        std::string msg = last_error_message();
        xpir_server_destroy(sv);
        return fail(rc, msg);
    }
    *out = sv;
    return XPIR_OK;
}

int xpir_server_destroy(xpir_server* sv) {
    if (!sv) return XPIR_OK;
    for (auto& e : sv->ring) xpir_store_destroy(e.st);
    for (auto& e : sv->retired) xpir_store_destroy(e.st);
    for (auto* st : sv->spare) xpir_store_destroy(st);
    xpir_table_destroy(sv->table);
    xpir_window_destroy(sv->window);
    delete sv;
    return XPIR_OK;
}

int xpir_server_apply_round(xpir_server* sv, const uint32_t* beta1, const uint32_t* beta2, const uint8_t* payload,
                            const uint32_t* interest, uint32_t h_per_write, uint64_t n, int seal_after,
                            uint32_t* reports, uint64_t* sealed_epoch) {
    return xpir_server_apply_round_sharded(sv, beta1, beta2, payload, interest, h_per_write, n, seal_after, nullptr,
                                           nullptr, nullptr, reports, sealed_epoch);
}

// The table insert of a round on a payload shard: H2D, replicated walk, gather
// (peer shards), the caller's barrier, scatter.
static int table_insert_sharded(xpir_table* t, const uint32_t* b1, const uint32_t* b2, const uint8_t* payload,
                                uint64_t n, uint32_t* reports, const xpir_shard_map* map,
                                void (*barrier)(void*), void* ctx) {
    std::lock_guard<std::mutex> lk(t->mu);
    DeviceGuard g(t->device);
    cudaStream_t s = t->stream;
    XCK(t->in_b1.ensure(4 * n));
    XCK(t->in_b2.ensure(4 * n));
    XCK(t->in_payload.ensure(n * t->d.item));
    XCK(t->in_reports.ensure(16 * n));
    XCK(cudaMemcpyAsync(t->in_b1.p, b1, 4 * n, cudaMemcpyHostToDevice, s));
    XCK(cudaMemcpyAsync(t->in_b2.p, b2, 4 * n, cudaMemcpyHostToDevice, s));
    XCK(cudaMemcpyAsync(t->in_payload.p, payload, n * t->d.item, cudaMemcpyHostToDevice, s));
    // beta ranges were checked on the host (xpir_server_apply_round_sharded)
    int rc = table_walk_impl(t, t->in_b1.as<uint32_t>(), t->in_b2.as<uint32_t>(), n, t->in_reports.as<uint32_t>(), s);
    if (!rc) rc = xpir_table_apply_gather_dev(t, map, s);
    if (rc) return rc;
    XCK(cudaStreamSynchronize(s));
    if (barrier) barrier(ctx);  // every shard has staged what moves into its range
    rc = xpir_table_apply_scatter_dev(t, t->in_payload.as<uint8_t>(), s);
    if (rc) return rc;
    if (reports) XCK(cudaMemcpyAsync(reports, t->in_reports.p, 16 * n, cudaMemcpyDeviceToHost, s));
    XCK(cudaStreamSynchronize(s));
    return XPIR_OK;
}

int xpir_server_apply_round_sharded(xpir_server* sv, const uint32_t* beta1, const uint32_t* beta2,
                                    const uint8_t* payload, const uint32_t* interest, uint32_t h_per_write,
                                    uint64_t n, int seal_after, const xpir_shard_map* map,
                                    void (*barrier)(void*), void* barrier_ctx, uint32_t* reports,
                                    uint64_t* sealed_epoch) {
    if (!sv) return fail(XPIR_EINVAL, "server_apply: null server");
    if (sv->table->sharded() && (!map || !barrier))
        return fail(XPIR_EINVAL, "server_apply: a payload shard needs the shard map and a barrier");
    if (sealed_epoch) *sealed_epoch = 0;
    if (n && (!beta1 || !beta2 || !payload || (h_per_write && !interest)))
        return fail(XPIR_EINVAL, "server_apply: null buffer");
    std::lock_guard<std::mutex> lk(sv->mu);
    // apply_write (server.cpp:58-73) for writes in order. Both precondition checks
    // are resolved on the host first, so the device work is exactly the reference's:
    //  * write kb with a bucket out of range throws before any state change
    //    (server.cpp:60-61): writes [0, kb) are applied;
    //  * write kp with an interest position >= m is inserted, its positions before
    //    the bad one are absorbed, then absorb throws (notify.cpp:62) and the write
    //    is not counted.
    const uint32_t m_bits = sv->window->m;
    uint64_t kb = n, kp = n, jp = 0;
    for (uint64_t k = 0; k < n && kb == n; ++k)
        if (beta1[k] >= sv->table->d.buckets || beta2[k] >= sv->table->d.buckets) kb = k;
    for (uint64_t k = 0; k < kb && kp == n; ++k)
        for (uint32_t j = 0; j < h_per_write; ++j)
            if (interest[k * h_per_write + j] >= m_bits) {
                kp = k;
                jp = j;
                break;
            }
    const uint64_t n_ins = kp < kb ? kp + 1 : kb;  // writes that reach Table::insert
    const uint64_t ok = kp < kb ? kp : kb;         // writes that complete
    if (n_ins) {
        int rc = sv->table->sharded()
                     ? table_insert_sharded(sv->table, beta1, beta2, payload, n_ins, reports, map, barrier,
                                            barrier_ctx)
                     : xpir_table_insert_batch(sv->table, beta1, beta2, payload, n_ins, reports);
        if (rc) return rc;
        // interest positions per rotation segment, then rotate (server.cpp:64-70)
        uint64_t a = 0;
        while (a < ok) {
            const uint64_t to_rot = sv->rotate_writes - (sv->writes % sv->rotate_writes);
            const uint64_t b = std::min(ok, a + to_rot);
            if (h_per_write) {
                rc = window_absorb_prechecked(sv->window, interest + a * h_per_write, (b - a) * h_per_write);
                if (rc) return rc;
            }
            sv->writes += b - a;
            if (sv->writes % sv->rotate_writes == 0) {
                rc = xpir_window_rotate(sv->window);
                if (rc) return rc;
            }
            a = b;
        }
        if (kp < kb) {
            rc = window_absorb_prechecked(sv->window, interest + kp * h_per_write, jp);
            if (rc) return rc;
            return fail(XPIR_EINVAL, "Window: position out of range");
        }
    }
    if (kb < n) return fail(XPIR_EINVAL, "write targets a bucket outside the table");
    if (seal_after) return server_seal(sv, sealed_epoch);
    return XPIR_OK;
}

int xpir_server_reserve(xpir_server* sv, uint64_t max_batch) {
    if (!sv) return fail(XPIR_EINVAL, "server_reserve: null server");
    std::lock_guard<std::mutex> lk(sv->mu);
    int rc = xpir_table_reserve(sv->table, max_batch);
    if (rc) return rc;
    xpir_table* t = sv->table;
    while (sv->ring.size() + sv->spare.size() < sv->epoch_ring) {
        xpir_store* st = nullptr;
        rc = xpir_store_create(sv->device, t->d.buckets, uint32_t(t->d.depth * t->d.item), t->lo, t->hi, &st);
        if (rc) return rc;
        sv->spare.push_back(st);
    }
    return XPIR_OK;
}

int xpir_server_seal(xpir_server* sv, uint64_t* epoch) {
    if (!sv) return fail(XPIR_EINVAL, "server_seal: null server");
    std::lock_guard<std::mutex> lk(sv->mu);
    return server_seal(sv, epoch);
}

int xpir_server_snapshot(xpir_server* sv, uint64_t epoch, xpir_store** st) {  // server.cpp:83-91
    if (!sv || !st) return fail(XPIR_EINVAL, "server_snapshot: null argument");
    std::lock_guard<std::mutex> lk(sv->mu);
    *st = nullptr;
    if (epoch == 0) epoch = sv->latest_epoch;
    for (auto& e : sv->ring)
        if (e.epoch == epoch) *st = e.st;
    return *st ? XPIR_OK : fail(XPIR_EINVAL, "server_snapshot: epoch not in the ring");
}

int xpir_server_snapshot_acquire(xpir_server* sv, uint64_t epoch, xpir_store** st, uint64_t* epoch_out) {
    if (!sv || !st) return fail(XPIR_EINVAL, "server_snapshot_acquire: null argument");
    std::lock_guard<std::mutex> lk(sv->mu);
    *st = nullptr;
    if (epoch == 0) epoch = sv->latest_epoch;
    for (auto& e : sv->ring)
        if (e.epoch == epoch) {
            e.pins += 1;
            *st = e.st;
            if (epoch_out) *epoch_out = e.epoch;
            return XPIR_OK;
        }
    return fail(XPIR_EINVAL, "server_snapshot_acquire: epoch not in the ring");
}

int xpir_server_snapshot_release(xpir_server* sv, xpir_store* st) {
    if (!sv || !st) return fail(XPIR_EINVAL, "server_snapshot_release: null argument");
    std::lock_guard<std::mutex> lk(sv->mu);
    for (auto& e : sv->ring)
        if (e.st == st && e.pins) {
            e.pins -= 1;
            return XPIR_OK;
        }
    for (size_t k = 0; k < sv->retired.size(); ++k)
        if (sv->retired[k].st == st && sv->retired[k].pins) {
            if (--sv->retired[k].pins == 0) {
                sv->spare.push_back(st);  // no epoch any more: the next seal copies it whole
                sv->retired.erase(sv->retired.begin() + long(k));
            }
            return XPIR_OK;
        }
    return fail(XPIR_EINVAL, "server_snapshot_release: store is not pinned");
}

// ServerCore::make_freeze (server.cpp:45-56): the deltas that will never change
// again (all but the newest) — base, newest index, digest over them, and their
// count; delta k's wire bytes come from xpir_window_encode_delta(window, k, ...).
int xpir_server_freeze(xpir_server* sv, uint64_t* base, uint64_t* newest, uint8_t digest[32], uint64_t* count) {
    if (!sv || !base || !newest || !digest || !count) return fail(XPIR_EINVAL, "server_freeze: null argument");
    std::lock_guard<std::mutex> lk(sv->mu);
    xpir_window* w = sv->window;
    const uint64_t size = w->deltas.size();
    *base = w->base;
    *newest = w->base + size - 2;  // window.newest() - 1
    *count = size - 1;
    return xpir_window_digest_n(w, size - 1, digest);
}

int xpir_server_info(xpir_server* sv, uint64_t* writes, uint64_t* latest_epoch, uint64_t* oldest_epoch,
                     xpir_table** table, xpir_window** window) {
    if (!sv) return fail(XPIR_EINVAL, "server_info: null server");
    std::lock_guard<std::mutex> lk(sv->mu);
    if (writes) *writes = sv->writes;
    if (latest_epoch) *latest_epoch = sv->latest_epoch;
    if (oldest_epoch) *oldest_epoch = sv->ring.empty() ? 0 : sv->ring.front().epoch;
    if (table) *table = sv->table;
    if (window) *window = sv->window;
    return XPIR_OK;
}

}  // extern "C"

