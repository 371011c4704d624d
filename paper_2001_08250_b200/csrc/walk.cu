// K6 (warp-cooperative): the cuckoo insertion walk of a write round, exact
// cuckoo::Table::insert semantics (cuckoo.cpp:56-126), one warp.
//
// The reference processes inserts one at a time. Most inserts are "simple": a
// free slot exists in beta1 or beta2 (cuckoo.cpp:73-84), no FIFO GC is due
// (:64-69) and no draw is consumed. For 32 consecutive inserts the warp
// decides in parallel which of them can be applied at once:
//   * lane k is simple in the pre-batch state, and
//   * no earlier lane j < k of the batch places into b1_k or b2_k (checked
//     with a small shared hash of placement buckets; a hash collision only
//     makes the check conservative), and
//   * no GC is due (live + k < capacity) and the FIFO ring has room.
// Then insert k sees exactly the pre-batch occupancy of its two buckets, so
// its outcome (lowest free slot of beta1, else of beta2) and its stamp
// (next_stamp + k) are what the sequential loop would produce. The longest
// prefix of such lanes is applied in parallel; the first lane that fails runs
// the sequential path (GC, eviction walk with DetRng draws) with the whole warp
// executing it redundantly (identical values in every lane: no broadcasts, and
// redundant stores of identical values to one address are benign), then the
// next batch starts right after it.
//
// Occupancy and "touched this round" bitmaps live in shared memory, as do the
// staged beta pairs and a 4096-entry ring of precomputed DetRng draws that the
// warp refills from the global draw window (DetRng::fill(8) per Rng::uniform
// draw, rng.cpp:9-31) between inserts, so the kernel only returns to the host
// when the global window (64 Ki draws) is exhausted.
// Payload bytes are not moved here: each touched slot records where its final
// content comes from (origin, see k_cuckoo_walk) for the gather/scatter kernels.
#include <cuda_runtime.h>

#include <cstdint>

#include "scan.cuh"

namespace xpir {

namespace {

constexpr uint32_t W_RING = 4096;      // staged draws (power of two)
constexpr uint32_t W_NEED = 640;       // draws that must be staged before a sequential insert (>= 501)
constexpr uint32_t W_CHUNK = 2048;     // staged inserts (beta pairs)
constexpr uint32_t W_HT = 1024;        // placement-bucket hash (power of two)
constexpr uint32_t FULL = 0xffffffffu;

}  // namespace

constexpr uint32_t WALKW_MAX_SLOTS = 64 * 1024 * 8;  // bit-packed maps: 64 KiB each

size_t walk_w_smem_bytes(uint64_t slots) {
    const size_t words = (slots + 31) / 32;
    return (2 * words) * 4 + W_RING * 8 + 2 * W_CHUNK * 4 + W_HT * 4 + 16;
}

// G == false: occupancy and touched maps bit-packed in shared memory (tables up to
// WALKW_MAX_SLOTS). G == true: any table size — occupancy read from the global
// `used` bytes (one 4/8-byte load per bucket for depth 4/8) and the touched set
// kept as touched_mark[slot] == batch id, as k_cuckoo_walk_x does; nothing is
// staged or written back.
// DEP != 0: the bucket depth as a compile-time constant (the depth-4 tables of
// every BASELINE config) — no run-time depth dispatch or multiplies per hop.
template <bool G, uint32_t DEP>
__global__ void __launch_bounds__(256, 1)
k_cuckoo_walk_w(CuckooDev d, CuckooState* __restrict__ gst, const uint32_t* __restrict__ beta1,
                const uint32_t* __restrict__ beta2, uint64_t i0, uint64_t n, uint32_t* __restrict__ reports) {
    if (!walk_prologue(gst, i0, n)) return;
    extern __shared__ __align__(16) uint32_t sm[];
    const uint32_t slots = G ? 0u : d.buckets * (DEP ? DEP : d.depth);
    const uint32_t words = (slots + 31) / 32;
    uint64_t* ring = reinterpret_cast<uint64_t*>(sm);  // 8-byte aligned first
    uint32_t* used_bits = sm + 2 * W_RING;
    uint32_t* touch_bits = used_bits + words;
    uint32_t* sb1 = touch_bits + words;
    uint32_t* sb2 = sb1 + W_CHUNK;
    uint32_t* htag = sb2 + W_CHUNK;

    CuckooState s = *gst;
    // stage the occupancy map and the touched map of this round
    for (uint32_t w = threadIdx.x; w < words; w += blockDim.x) {  // (G: words == 0)
        uint32_t v = 0;
        for (uint32_t b = 0; b < 32; ++b) {
            const uint32_t f = w * 32 + b;
            if (f < slots && d.used[f]) v |= 1u << b;
        }
        used_bits[w] = v;
        touch_bits[w] = 0;
    }
    for (uint32_t k = threadIdx.x; k < W_HT; k += blockDim.x) htag[k] = FULL;
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < (G ? 0u : s.n_touched); k += blockDim.x) {
        const uint32_t f = d.touched[k];
        atomicOr(&touch_bits[f >> 5], 1u << (f & 31));
    }
    __syncthreads();

    if (threadIdx.x < 32) {
        const uint32_t lane = threadIdx.x;
        const uint32_t depth = DEP ? DEP : d.depth;
        const uint32_t dmask = depth >= 32 ? FULL : (1u << depth) - 1u;  // depth <= 32 (launcher)
        const uint64_t fmask = d.fifo_cap - 1;
        const uint64_t gend = s.draw_base + s.draw_count;  // end of the global draw window
        uint64_t dr_hi = s.rng_block;                       // draws staged in the ring: [.., dr_hi)
        s.status = 0;

        auto free_mask = [&](uint32_t b) -> uint32_t {  // bit s set: slot s of bucket b is free
            if constexpr (G) {
                const uint8_t* u = d.used + size_t(b) * depth;
                if (depth == 4 || depth == 8) {  // 0/1 bytes -> one bit per slot
                    uint64_t w = depth == 4 ? uint64_t(*reinterpret_cast<const uint32_t*>(u))
                                            : *reinterpret_cast<const uint64_t*>(u);
                    w = (w | (w >> 7) | (w >> 14) | (w >> 21) | (w >> 28) | (w >> 35) | (w >> 42) | (w >> 49));
                    return uint32_t(~w) & dmask;  // bit k of byte 0 = used[k] (bytes are 0/1)
                }
                uint32_t m = 0;
                for (uint32_t k = 0; k < depth; ++k) m |= u[k] ? 0u : (1u << k);
                return m;
            }
            const uint32_t f0 = b * depth, w0 = f0 >> 5, sh = f0 & 31;
            uint64_t bits = used_bits[w0];
            if (sh + depth > 32) bits |= uint64_t(used_bits[w0 + 1]) << 32;
            return uint32_t(~(bits >> sh)) & dmask;
        };
        auto refill = [&]() {  // stage draws up to rng_block + W_RING (never past the window)
            uint64_t hi = s.rng_block + W_RING;
            if (hi > gend) hi = gend;
            for (uint64_t k = dr_hi + lane; k < hi; k += 32) ring[k & (W_RING - 1)] = d.draws[k - s.draw_base];
            dr_hi = hi > dr_hi ? hi : dr_hi;
            __syncwarp();
        };
        // ---- the sequential path (warp-redundant) ------------------------------
        auto is_touched = [&](uint32_t f) -> bool {
            if constexpr (G) return d.touched_mark[f] == s.batch_id;
            return (touch_bits[f >> 5] >> (f & 31)) & 1u;
        };
        auto touch = [&](uint32_t f, int64_t org) {
            if (!is_touched(f)) {
                if constexpr (G) d.touched_mark[f] = s.batch_id;
                else touch_bits[f >> 5] |= 1u << (f & 31);
                d.touched[s.n_touched++] = f;
            }
            d.origin[f] = org;
        };
        auto place = [&](uint32_t f, uint32_t b1, uint32_t b2, uint64_t stamp, int64_t org) {  // :37-46
            if constexpr (G) d.used[f] = 1;
            else used_bits[f >> 5] |= 1u << (f & 31);
            d.beta1[f] = b1;
            d.beta2[f] = b2;
            d.stamp[f] = stamp;
            d.fifo[stamp & fmask] = int64_t(f);
            touch(f, org);
            s.live++;
        };
        auto clear = [&](uint32_t f) {  // :48-54
            if constexpr (G) d.used[f] = 0;
            else used_bits[f >> 5] &= ~(1u << (f & 31));
            d.fifo[d.stamp[f] & fmask] = -1;
            d.beta1[f] = 0;
            d.beta2[f] = 0;
            d.stamp[f] = 0;
            touch(f, -1);
            s.live--;
        };
        auto uniform = [&](uint64_t bound) -> uint64_t {  // rng.cpp:9-16 over staged DetRng::fill(8) draws
            if ((bound & (bound - 1)) == 0) return ring[(s.rng_block++) & (W_RING - 1)] & (bound - 1);
            const uint64_t tail = (~uint64_t(0) % bound + 1) % bound;
            for (;;) {
                const uint64_t v = ring[(s.rng_block++) & (W_RING - 1)];
                if (tail == 0 || v <= ~uint64_t(0) - tail) return v % bound;
            }
        };
        // returns false when the insert could not run (status set)
        auto insert_one = [&](uint64_t i, uint32_t b1, uint32_t b2) -> bool {
            if (dr_hi - s.rng_block < W_NEED) {
                refill();
                if (dr_hi - s.rng_block < W_NEED) {
                    s.status = 1;  // host refills the global window from nonce rng_block, resumes at i
                    return false;
                }
            }
            // FIFO ring room for this insert's stamp, checked before any state changes
            // (stamps of dead entries at the head never matter again: skip them); on
            // overflow the host grows the ring and resumes at this insert
            if (s.next_stamp - s.fifo_head >= d.fifo_cap) {
                while (s.fifo_head < s.next_stamp && d.fifo[s.fifo_head & fmask] < 0) s.fifo_head++;
                if (s.next_stamp - s.fifo_head >= d.fifo_cap) {
                    s.status = 2;
                    return false;
                }
            }
            uint32_t stored = 0, dropped = 0, gc = 0, disp = 0;
            // both buckets' occupancy in one round trip, together with the FIFO head
            // reads below (re-read when the GC frees a slot)
            uint32_t m1 = free_mask(b1), m2 = free_mask(b2);
            s.writes++;  // :62
            if (s.live == d.capacity) {  // :64-69 FIFO GC of the oldest entry
                while (d.fifo[s.fifo_head & fmask] < 0) s.fifo_head++;
                clear(uint32_t(d.fifo[s.fifo_head & fmask]));
                gc = 1;
                m1 = free_mask(b1);
                m2 = free_mask(b2);
            }
            const uint64_t stamp = s.next_stamp++;  // :71 (ring room checked above)
            if (m1) m2 = 0;  // :73-84 (bucket 2 only when bucket 1 is full)
            if (m1 | m2) {
                const uint32_t b = m1 ? b1 : b2;
                place(b * depth + uint32_t(__ffs(int(m1 ? m1 : m2)) - 1), b1, b2, stamp, int64_t(i));
                stored = 1;
            } else {  // :86-125 random-walk eviction
                uint32_t be = uniform(2) == 0 ? b1 : b2;
                uint32_t c1 = b1, c2 = b2;
                uint64_t cst = stamp;
                int64_t corg = int64_t(i);
                bool carry_incoming = true, incoming_stored = false, done = false;
                // power-of-two depth: the victim slot is the next staged draw, so its
                // metadata is loaded together with the bucket's occupancy (unused when
                // the bucket has room) — one dependent round trip per hop
                const bool spec = (depth & (depth - 1)) == 0;
                for (uint32_t hops = 0;; ++hops) {
                    uint32_t vs = 0, v1 = 0, v2 = 0, vtm = 0;
                    uint64_t vst = 0;
                    int64_t vo = 0;
                    if (spec) {
                        vs = uint32_t(ring[s.rng_block & (W_RING - 1)]) & (depth - 1);
                        const uint32_t vf = be * depth + vs;
                        v1 = d.beta1[vf];
                        v2 = d.beta2[vf];
                        vst = d.stamp[vf];
                        vo = d.origin[vf];
                        if constexpr (G) vtm = d.touched_mark[vf];
                    }
                    const uint32_t fm = free_mask(be);
                    if (fm) {
                        place(be * depth + uint32_t(__ffs(int(fm)) - 1), c1, c2, cst, corg);
                        if (carry_incoming) incoming_stored = true;
                        stored = incoming_stored;
                        disp = hops;
                        done = true;
                        break;
                    }
                    if (hops == XPIR_MAX_DISPLACEMENTS_DEV) break;
                    if (spec) {
                        s.rng_block++;  // == uniform(depth) for a power-of-two bound
                    } else {
                        vs = uint32_t(uniform(depth));
                        const uint32_t vf = be * depth + vs;
                        v1 = d.beta1[vf];
                        v2 = d.beta2[vf];
                        vst = d.stamp[vf];
                        vo = d.origin[vf];
                        if constexpr (G) vtm = d.touched_mark[vf];
                    }
                    const uint32_t vf = be * depth + vs;
                    bool vt;
                    if constexpr (G) vt = vtm == s.batch_id;
                    else vt = is_touched(vf);
                    const int64_t vorg = vt ? vo : -int64_t(vf) - 2;
                    // clear(vf) then place(vf, carry) (:110-113): occupancy and live unchanged
                    d.fifo[vst & fmask] = -1;
                    d.beta1[vf] = c1;
                    d.beta2[vf] = c2;
                    d.stamp[vf] = cst;
                    d.fifo[cst & fmask] = int64_t(vf);
                    if (!vt) {  // touch(vf, corg)
                        if constexpr (G) d.touched_mark[vf] = s.batch_id;
                        else touch_bits[vf >> 5] |= 1u << (vf & 31);
                        d.touched[s.n_touched++] = vf;
                    }
                    d.origin[vf] = corg;
                    if (carry_incoming) incoming_stored = true;
                    c1 = v1;
                    c2 = v2;
                    cst = vst;
                    corg = vorg;
                    carry_incoming = false;
                    be = v1 == be ? v2 : v1;  // :118
                }
                if (!done) {  // :122-125
                    disp = XPIR_MAX_DISPLACEMENTS_DEV;
                    dropped = 1;
                    stored = incoming_stored;
                }
            }
            if (reports && lane == 0) reinterpret_cast<uint4*>(reports)[i] = make_uint4(stored, dropped, gc, disp);
            return true;
        };

        uint64_t c = i0;
        bool stop = false;
        while (c < n && !stop) {
            // stage the next chunk of beta pairs
            const uint64_t c0 = c;
            const uint32_t cn = uint32_t((n - c0) < W_CHUNK ? (n - c0) : W_CHUNK);
            for (uint32_t k = lane; k < cn; k += 32) {
                sb1[k] = beta1[c0 + k];
                sb2[k] = beta2[c0 + k];
            }
            __syncwarp();
            const uint64_t ce = c0 + cn;
            while (c < ce) {
                // ---- parallel batch of simple inserts ---------------------------
                const uint32_t avail = uint32_t((ce - c) < 32 ? (ce - c) : 32);
                const bool valid = lane < avail;
                const uint32_t b1 = valid ? sb1[c - c0 + lane] : 0u, b2 = valid ? sb2[c - c0 + lane] : 0u;
                const uint32_t m1 = valid ? free_mask(b1) : 0u, m2 = valid ? free_mask(b2) : 0u;
                const bool simple = (m1 | m2) != 0;
                const uint32_t pb = m1 ? b1 : b2, pm = m1 ? m1 : m2;
                if (simple) atomicMin(&htag[pb & (W_HT - 1)], lane);
                __syncwarp();
                const bool conflict = valid && (htag[b1 & (W_HT - 1)] < lane || htag[b2 & (W_HT - 1)] < lane);
                __syncwarp();
                if (simple) htag[pb & (W_HT - 1)] = FULL;
                const uint64_t room_gc = d.capacity - s.live;
                const uint64_t room_fifo = d.fifo_cap - (s.next_stamp - s.fifo_head);
                const bool halt = !simple || conflict || lane >= room_gc || lane >= room_fifo;
                const uint32_t hm = __ballot_sync(FULL, halt);
                const uint32_t L = hm ? uint32_t(__ffs(int(hm)) - 1) : 32u;
                bool newt = false;
                uint32_t f = 0;
                if (lane < L) {
                    const uint64_t i = c + lane;
                    f = pb * depth + uint32_t(__ffs(int(pm)) - 1);
                    const uint64_t stamp = s.next_stamp + lane;
                    if constexpr (G) d.used[f] = 1;
                    else atomicOr(&used_bits[f >> 5], 1u << (f & 31));
                    d.beta1[f] = b1;
                    d.beta2[f] = b2;
                    d.stamp[f] = stamp;
                    d.fifo[stamp & fmask] = int64_t(f);
                    d.origin[f] = int64_t(i);
                    newt = !is_touched(f);
                    if (newt) {
                        if constexpr (G) d.touched_mark[f] = s.batch_id;
                        else atomicOr(&touch_bits[f >> 5], 1u << (f & 31));
                    }
                    if (reports) reinterpret_cast<uint4*>(reports)[i] = make_uint4(1, 0, 0, 0);
                }
                const uint32_t nm = __ballot_sync(FULL, newt);
                if (newt) d.touched[s.n_touched + __popc(nm & ((1u << lane) - 1u))] = f;
                s.n_touched += __popc(nm);
                s.writes += L;
                s.live += L;
                s.next_stamp += L;
                c += L;
                __syncwarp();
                // ---- the first lane that could not go in parallel ---------------
                if (L < 32 && c < ce) {
                    const uint32_t k = uint32_t(c - c0);
                    if (!insert_one(c, sb1[k], sb2[k])) {
                        stop = true;
                        break;
                    }
                    ++c;
                    __syncwarp();
                }
            }
        }
        s.resume_at = c;
        if (lane == 0) *gst = s;
    }
    __syncthreads();
    // occupancy map back to the global byte array (G: words == 0)
    for (uint32_t w = threadIdx.x; w < words; w += blockDim.x) {
        const uint32_t v = used_bits[w];
        const uint32_t f0 = w * 32;
        for (uint32_t k = 0; k < 32 && f0 + k < slots; ++k) d.used[f0 + k] = (v >> k) & 1u;
    }
}

cudaError_t launch_cuckoo_walk_w(const CuckooDev& d, CuckooState* st, const uint32_t* beta1, const uint32_t* beta2,
                                 uint64_t i0, uint64_t n, uint32_t* reports, cudaStream_t s, bool force_global) {
    const uint64_t slots = uint64_t(d.buckets) * d.depth;
    const bool g = force_global || slots > WALKW_MAX_SLOTS;
    const size_t smem = walk_w_smem_bytes(g ? 0 : slots);
    auto k = d.depth == 4 ? (g ? k_cuckoo_walk_w<true, 4> : k_cuckoo_walk_w<false, 4>)
                          : (g ? k_cuckoo_walk_w<true, 0> : k_cuckoo_walk_w<false, 0>);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    k<<<1, 256, smem, s>>>(d, st, beta1, beta2, i0, n, reports);
    return cudaGetLastError();
}

bool walk_w_supported(const CuckooDev& d) {
    // the global-map variant takes any size; slot ids stay 32-bit
    return uint64_t(d.buckets) * d.depth < (uint64_t(1) << 32) && d.depth <= 32;
}

}  // namespace xpir
