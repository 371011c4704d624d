// K6x: the cuckoo insertion walk with the eviction control flow entirely on chip
// (exact cuckoo::Table::insert semantics, cuckoo.cpp:56-126), one warp.
//
// An eviction hop needs only three things to decide the next hop: the occupancy
// of the current bucket (is there a free slot?), the next DetRng draw (which
// slot to evict) and the victim's alternate bucket. The last one is
// beta1 ^ beta2 ^ be, so the walk keeps alt[slot] = beta1 ^ beta2 (16 bits,
// buckets <= 65,536) for every slot on chip: the first 98,304 slots in shared
// memory, the rest (up to 32,768 more) in the walking warp's Tensor Memory lane
// quadrant (32 lanes x 512 columns x 32 bits = two 16-bit entries per column
// cell, tcgen05.ld/st .32x32b.x1 + a shuffle). A hop is then a handful of
// on-chip accesses instead of one dependent L2 round trip (k_cuckoo_walk_w).
//
// The data that moves along the chain (beta1, beta2, stamp, payload origin of
// each displaced item) is resolved after the chain in one parallel step: the
// chain's slots v_0..v_{h-1} are logged; the item carried out of hop k is the
// content of v_k at that time, i.e. the pre-chain content of v_k unless v_k was
// visited earlier in the chain at step i, in which case it is whatever was
// placed at step i. For chains of up to 32 hops (nearly all) lane k loads the
// pre-chain content of v_k while the walk goes on (the global metadata is not
// written during the walk), revisits are found with one __match_any_sync, each
// placement's source by a few rounds of shuffles, and lanes write the final
// content of every slot (its last visit), its FIFO entry (an item's entry is its
// final slot, or -1 if it was dropped) and its touched mark. Longer chains take
// the same steps through a global scratch array.
//
// Simple inserts (a free slot in beta1 or beta2) are applied 32 at a time as in
// k_cuckoo_walk_w. The touched set is kept as touched_mark[slot] == batch id in
// global memory (written, never read on a hot path) and the touched list is
// rebuilt from it by the whole CTA at the end of the launch.
#include <cuda_runtime.h>

#include <cstdint>

#include "scan.cuh"

namespace xpir {

namespace {

constexpr uint32_t X_SM_SLOTS = 98304;   // alt entries in shared memory
constexpr uint32_t X_TM_SLOTS = 32768;   // alt entries in TMEM (lanes 0-31, 512 columns, 2 per cell)
constexpr uint32_t X_RING = 1024;        // staged draws
constexpr uint32_t X_NEED = 640;         // draws staged before a sequential insert (>= 501)
constexpr uint32_t X_CHUNK = 256;        // staged inserts (beta pairs)
constexpr uint32_t X_HT = 256;           // placement-bucket hash of the batch path
constexpr uint32_t X_CHAIN = 512;        // >= MAX_DISPLACEMENTS + 1
constexpr uint32_t X_HS = 1000;          // long-chain slot -> last-visit hash (>= 2 x distinct slots)
constexpr uint32_t X_EMPTY = 0xffffffffu;
constexpr uint32_t FULLM = 0xffffffffu;
constexpr uint16_t NONE16 = 0xffff;

// A finished chain handed from the walking warp to the resolving warp: its slots
// (chains of <= 32 hops; longer ones stay in the shared chain[] log), final slot
// (FULLM = dropped) and the incoming item.
struct XRec {
    uint32_t v[32];
    uint32_t h, final_slot, b1, b2;
    uint64_t stamp, i;
};

struct XLayout {
    uint32_t alt_sm, words;
    size_t o_ring, o_alt, o_used, o_sb1, o_sb2, o_ht, o_chain, o_hash, o_src, o_q, o_qf, o_taddr, total;
    __host__ __device__ explicit XLayout(uint32_t slots) {
        alt_sm = slots < X_SM_SLOTS ? slots : X_SM_SLOTS;
        words = (slots + 31) / 32;
        auto a16 = [](size_t x) { return (x + 15) & ~size_t(15); };  // every region 16-byte aligned
        o_ring = 0;
        o_alt = a16(o_ring + X_RING * 8);
        o_used = a16(o_alt + alt_sm * 2);
        o_sb1 = a16(o_used + words * 4);
        o_sb2 = a16(o_sb1 + X_CHUNK * 4);
        o_ht = a16(o_sb2 + X_CHUNK * 4);
        o_chain = a16(o_ht + X_HT * 4);
        o_hash = a16(o_chain + X_CHAIN * 4);  // u32 entries: slot << 9 | last visit index
        o_src = a16(o_hash + X_HS * 4);
        o_q = a16(o_src + (X_CHAIN + 16) * 2);  // 2 hand-off records (XRec)
        o_qf = a16(o_q + 2 * sizeof(XRec));    // flags: full[0], full[1], chain[] busy, done
        o_taddr = a16(o_qf + 16);
        total = o_taddr + 16;
    }
};

__device__ __forceinline__ uint32_t tm_ld1(uint32_t a) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(a));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" : "+r"(v)::"memory");
    return v;
}
// cp.async of 4 / 8 bytes: the prefetch does not hold any register scoreboard
template <int N>
__device__ __forceinline__ void cp_async_ca(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(dst), "l"(src), "n"(N) : "memory");
}
__device__ __forceinline__ void tm_st1(uint32_t a, uint32_t v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};\n" ::"r"(a), "r"(v));
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
}

}  // namespace

bool walk_x_supported(const CuckooDev& d) {
    const uint64_t slots = uint64_t(d.buckets) * d.depth;
    return slots <= X_SM_SLOTS + X_TM_SLOTS && d.buckets <= 65536 && d.depth <= 32 && d.chain_pre &&
           XLayout(uint32_t(slots)).total <= 232448;
}

// DEP != 0: compile-time bucket depth (4 at every BASELINE config).
template <uint32_t DEP>
__global__ void __launch_bounds__(256, 1)
k_cuckoo_walk_x(CuckooDev d, CuckooState* __restrict__ gst, const uint32_t* __restrict__ beta1,
                const uint32_t* __restrict__ beta2, uint64_t i0, uint64_t n, uint32_t* __restrict__ reports) {
    if (!walk_prologue(gst, i0, n)) return;
    extern __shared__ __align__(16) uint8_t smx[];
    const uint32_t slots = d.buckets * (DEP ? DEP : d.depth);
    const XLayout L(slots);
    uint64_t* ring = reinterpret_cast<uint64_t*>(smx + L.o_ring);
    uint16_t* alt = reinterpret_cast<uint16_t*>(smx + L.o_alt);
    uint32_t* used_bits = reinterpret_cast<uint32_t*>(smx + L.o_used);
    uint32_t* sb1 = reinterpret_cast<uint32_t*>(smx + L.o_sb1);
    uint32_t* sb2 = reinterpret_cast<uint32_t*>(smx + L.o_sb2);
    uint32_t* htag = reinterpret_cast<uint32_t*>(smx + L.o_ht);
    uint32_t* chain = reinterpret_cast<uint32_t*>(smx + L.o_chain);
    uint32_t* hsh = reinterpret_cast<uint32_t*>(smx + L.o_hash);
    uint16_t* srck = reinterpret_cast<uint16_t*>(smx + L.o_src);
    const uint32_t smem_base = static_cast<uint32_t>(__cvta_generic_to_shared(smx));
    const bool use_tm = slots > X_SM_SLOTS;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (use_tm && warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_base +
                                                                                              uint32_t(L.o_taddr)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    // stage occupancy and the alternate-bucket index of every slot
    for (uint32_t w = threadIdx.x; w < L.words; w += blockDim.x) {
        uint32_t v = 0;
        for (uint32_t b = 0; b < 32; ++b) {
            const uint32_t f = w * 32 + b;
            if (f < slots && d.used[f]) v |= 1u << b;
        }
        used_bits[w] = v;
    }
    for (uint32_t f = threadIdx.x; f < L.alt_sm; f += blockDim.x) alt[f] = uint16_t(d.beta1[f] ^ d.beta2[f]);
    for (uint32_t k = threadIdx.x; k < X_HT; k += blockDim.x) htag[k] = FULLM;
    if (threadIdx.x < 4) reinterpret_cast<volatile uint32_t*>(smx + L.o_qf)[threadIdx.x] = 0;
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tbase = use_tm ? *reinterpret_cast<const uint32_t*>(smx + L.o_taddr) : 0u;

    CuckooState s = *gst;
    const uint32_t depth = DEP ? DEP : d.depth;
    const uint64_t fmask = d.fifo_cap - 1;
    XRec* recs = reinterpret_cast<XRec*>(smx + L.o_q);
    volatile uint32_t* qflag = reinterpret_cast<volatile uint32_t*>(smx + L.o_qf);
    auto touch_store = [&](uint32_t f, int64_t org) {  // lane-local store of one slot's origin + mark
        d.origin[f] = org;
        d.touched_mark[f] = s.batch_id;
    };
    // ---- resolve a finished chain: who ends where (see the header comment); warp 1 ----
    auto resolve_chain = [&](const XRec& r) {
        const uint32_t h = r.h, final_slot = r.final_slot, b1 = r.b1, b2 = r.b2;
        const uint64_t stamp = r.stamp, i = r.i;
        if (h <= 32) {
            // ---- resolve a short chain in registers -------------------------
            // lane k holds chain[k] and its pre-chain content; revisits by match_any
            const uint32_t my_v = lane < h ? r.v[lane] : (0x80000000u | lane);
            uint64_t my_st = 0;
            int64_t my_org = 0;
            uint32_t my_b1 = 0, my_b2 = 0, my_mark = 0;
            if (lane < h) {
                my_st = d.stamp[my_v];
                my_org = d.origin[my_v];
                my_b1 = d.beta1[my_v];
                my_b2 = d.beta2[my_v];
                my_mark = d.touched_mark[my_v];
            }
            const int64_t my_pre_org = my_mark == s.batch_id ? my_org : -int64_t(my_v) - 2;
            const uint32_t mm = __match_any_sync(FULLM, my_v);
            const uint32_t below = mm & ((1u << lane) - 1u);
            const uint32_t above = mm & ~((2u << lane) - 1u);
            const int prev = below ? 31 - __clz(int(below)) : -1;  // last earlier visit
            // f(k) = the item carried out of hop k: the pre-content of chain[k] (= k),
            // or the item placed at its previous visit p (INC if p == 0, else f(p - 1))
            int cur = int(lane), res = -2;  // -2 pending, -1 incoming, j >= 0 pre(chain[j])
            bool pend = lane < h;
            if (!pend) res = int(lane);
            while (__any_sync(FULLM, pend)) {
                const int p = __shfl_sync(FULLM, prev, cur & 31);
                if (pend) {
                    if (p < 0) {
                        res = cur;
                        pend = false;
                    } else if (p == 0) {
                        res = -1;
                        pend = false;
                    } else {
                        cur = p - 1;
                    }
                }
            }
            // step k places item src(k) = (k == 0 ? incoming : f(k - 1)) at chain[k];
            // step h places f(h - 1) at the final slot (or drops it)
            const int srck_l = __shfl_up_sync(FULLM, res, 1);
            const int src_here = lane == 0 ? -1 : srck_l;
            const int src_final = h == 0 ? -1 : __shfl_sync(FULLM, res, (h - 1) & 31);
            auto content = [&](int src, uint32_t& c1, uint32_t& c2, uint64_t& cst, int64_t& corg) {
                const int sl = src < 0 ? 0 : src;
                const uint32_t x1 = __shfl_sync(FULLM, my_b1, sl), x2 = __shfl_sync(FULLM, my_b2, sl);
                const uint64_t xs = __shfl_sync(FULLM, my_st, sl);
                const int64_t xo = __shfl_sync(FULLM, my_pre_org, sl);
                if (src < 0) {
                    c1 = b1;
                    c2 = b2;
                    cst = stamp;
                    corg = int64_t(i);
                } else {
                    c1 = x1;
                    c2 = x2;
                    cst = xs;
                    corg = xo;
                }
            };
            uint32_t c1, c2;
            uint64_t cst;
            int64_t corg;
            content(src_here, c1, c2, cst, corg);
            if (lane < h && above == 0) {  // last visit of chain[lane]: its final content
                d.beta1[my_v] = c1;
                d.beta2[my_v] = c2;
                d.stamp[my_v] = cst;
                d.fifo[cst & fmask] = int64_t(my_v);
                touch_store(my_v, corg);
            }
            content(src_final, c1, c2, cst, corg);
            if (lane == 0) {
                if (final_slot == FULLM) {
                    d.fifo[cst & fmask] = -1;  // the dropped item leaves the FIFO
                } else {
                    d.beta1[final_slot] = c1;
                    d.beta2[final_slot] = c2;
                    d.stamp[final_slot] = cst;
                    d.fifo[cst & fmask] = int64_t(final_slot);
                    touch_store(final_slot, corg);
                }
            }
            __syncwarp();
        } else {
        // ---- resolve a long chain through global scratch ----------------
        // Chunks of 32 hops in order, O(h) overall: within a chunk revisits are
        // found with __match_any_sync, across chunks through a shared-memory hash
        // (slot -> last visit so far); srck[j] = the item placed at step j
        // (NONE16 = the incoming one, q = the pre-chain content of chain[q]).
        uint64_t* pre = d.chain_pre;  // [3 * X_CHAIN]: (b1 | b2 << 32), stamp, origin
        auto hslot = [](uint32_t v) { return (v * 2654435761u) % X_HS; };
        for (uint32_t k = lane; k < X_HS; k += 32) hsh[k] = X_EMPTY;
        if (lane == 0) srck[0] = NONE16;
        __syncwarp();
        for (uint32_t base = 0; base < h; base += 32) {
            const uint32_t k = base + lane;
            const bool valid = k < h;
            const uint32_t v = valid ? chain[k] : (0x80000000u | lane);
            if (valid) {
                pre[3 * k] = uint64_t(d.beta1[v]) | uint64_t(d.beta2[v]) << 32;
                pre[3 * k + 1] = d.stamp[v];
                const int64_t o = d.origin[v];
                pre[3 * k + 2] = uint64_t(d.touched_mark[v] == s.batch_id ? o : -int64_t(v) - 2);
            }
            const uint32_t mm = __match_any_sync(FULLM, v);
            const uint32_t below = mm & ((1u << lane) - 1u);
            const uint32_t above = mm & ~((2u << lane) - 1u);
            // last earlier visit: in this chunk, else from the hash (earlier chunks)
            int prev = below ? int(base) + 31 - __clz(int(below)) : -1;
            uint32_t hpos = hslot(v), hfound = X_EMPTY;
            if (valid && !below) {
                for (;;) {
                    const uint32_t e = hsh[hpos];
                    if (e == X_EMPTY) break;
                    if ((e >> 9) == v) {
                        hfound = hpos;
                        prev = int(e & 511u);
                        break;
                    }
                    hpos = hpos + 1 == X_HS ? 0 : hpos + 1;
                }
            }
            // f(k) = item carried out of hop k = srck[k + 1]:
            // prev < 0 -> k; else srck[prev] (known when prev <= base, else f(prev - 1) in this chunk)
            int cur = int(k), res = -3;  // -3 pending
            bool pend = valid;
            while (__any_sync(FULLM, pend)) {
                const int p = __shfl_sync(FULLM, prev, (cur - int(base)) & 31);
                if (pend) {
                    if (p < 0) {
                        res = cur;
                        pend = false;
                    } else if (p <= int(base)) {
                        res = srck[p] == NONE16 ? -1 : int(srck[p]);
                        pend = false;
                    } else {
                        cur = p - 1;
                    }
                }
            }
            if (valid) srck[k + 1] = res < 0 ? NONE16 : uint16_t(res);
            // record the last visit of each slot of this chunk
            if (valid && above == 0) {
                const uint32_t ent = v << 9 | k;
                if (hfound != X_EMPTY) {
                    hsh[hfound] = ent;
                } else {
                    uint32_t q = hslot(v);
                    for (;;) {
                        const uint32_t old = atomicCAS(&hsh[q], X_EMPTY, ent);
                        if (old == X_EMPTY) break;
                        if ((old >> 9) == v) {  // seen in an earlier chunk and earlier in this one
                            hsh[q] = ent;
                            break;
                        }
                        q = q + 1 == X_HS ? 0 : q + 1;
                    }
                }
            }
            __syncwarp();
        }
        for (uint32_t k = lane; k <= h; k += 32) {
            const uint16_t src = srck[k];
            uint32_t slot;
            if (k < h) {
                slot = chain[k];
                uint32_t q = hslot(slot), e;
                while ((e = hsh[q]) >> 9 != slot) q = q + 1 == X_HS ? 0 : q + 1;
                if ((e & 511u) != k) continue;  // not the last visit of this slot
            } else {
                slot = final_slot;
            }
            uint32_t c1 = b1, c2 = b2;
            uint64_t cst = stamp;
            int64_t corg = int64_t(i);
            if (src != NONE16) {
                const uint64_t bb = pre[3 * src];
                c1 = uint32_t(bb);
                c2 = uint32_t(bb >> 32);
                cst = pre[3 * src + 1];
                corg = int64_t(pre[3 * src + 2]);
            }
            if (slot == FULLM) {  // the dropped item leaves the FIFO
                d.fifo[cst & fmask] = -1;
                continue;
            }
            d.beta1[slot] = c1;
            d.beta2[slot] = c2;
            d.stamp[slot] = cst;
            d.fifo[cst & fmask] = int64_t(slot);
            touch_store(slot, corg);
        }
        __syncwarp();
        }
            };
    if (warp == 0) {
        const uint32_t dmask = depth >= 32 ? FULLM : (1u << depth) - 1u;
        const bool dpow2 = (depth & (depth - 1)) == 0;
        const uint64_t gend = s.draw_base + s.draw_count;
        uint64_t dr_hi = s.rng_block;
        s.status = 0;
        if (use_tm) {  // TMEM part of alt: column c, lane l holds slots X_SM + 64c + 2l (+1)
            for (uint32_t c0 = 0; c0 < 512; c0 += 8) {  // 8 columns per store, loads issued together
                uint32_t v[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t f = X_SM_SLOTS + (c0 + k) * 64 + 2 * lane;
                    v[k] = 0;
                    if (f < slots) v[k] = (d.beta1[f] ^ d.beta2[f]) & 0xffffu;
                    if (f + 1 < slots) v[k] |= ((d.beta1[f + 1] ^ d.beta2[f + 1]) & 0xffffu) << 16;
                }
                asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(tbase + c0),
                             "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
            }
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        }
        // alt[] accessor (warp-uniform slot for the TMEM path):
        // returns the old value and stores x (one read-modify-write)
        auto alt_swap = [&](uint32_t f, uint32_t x) -> uint32_t {
            if (f < X_SM_SLOTS) {
                const uint32_t old = alt[f];
                alt[f] = uint16_t(x);
                return old;
            }
            const uint32_t i = f - X_SM_SLOTS, col = tbase + (i >> 6), ln = (i >> 1) & 31, hi = i & 1;
            __syncwarp();  // .sync.aligned TMEM access: the warp must be converged
            uint32_t cell = tm_ld1(col);
            const uint32_t v = __shfl_sync(FULLM, cell, ln);
            if (lane == ln) cell = hi ? (cell & 0xffffu) | (x << 16) : (cell & 0xffff0000u) | (x & 0xffffu);
            tm_st1(col, cell);
            return hi ? v >> 16 : v & 0xffffu;
        };
        auto free_mask = [&](uint32_t b) -> uint32_t {
            const uint32_t f0 = b * depth, w0 = f0 >> 5, sh = f0 & 31;
            uint64_t bits = used_bits[w0];
            if (sh + depth > 32) bits |= uint64_t(used_bits[w0 + 1]) << 32;
            return uint32_t(~(bits >> sh)) & dmask;
        };
        auto refill = [&]() {
            uint64_t hi = s.rng_block + X_RING;
            if (hi > gend) hi = gend;
            for (uint64_t k = dr_hi + lane; k < hi; k += 32) ring[k & (X_RING - 1)] = d.draws[k - s.draw_base];
            dr_hi = hi > dr_hi ? hi : dr_hi;
            __syncwarp();
        };
        auto uniform = [&](uint64_t bound) -> uint64_t {  // rng.cpp:9-16
            if ((bound & (bound - 1)) == 0) return ring[(s.rng_block++) & (X_RING - 1)] & (bound - 1);
            const uint64_t tail = (~uint64_t(0) % bound + 1) % bound;
            for (;;) {
                const uint64_t v = ring[(s.rng_block++) & (X_RING - 1)];
                if (tail == 0 || v <= ~uint64_t(0) - tail) return v % bound;
            }
        };
        // hand-off to warp 1: record slots alternate; flags are written after a fence
        uint32_t wslot = 0;
        auto wait_zero = [&](uint32_t k) {
            while (qflag[k] != 0) __nanosleep(20);
            __syncwarp();
            __threadfence_block();
        };
        auto drain = [&]() {  // every handed-off chain resolved (its metadata written)
            wait_zero(0);
            wait_zero(1);
            wait_zero(2);
        };

        // the sequential path (warp-redundant: every lane runs it with the same values)
        auto insert_one = [&](uint64_t i, uint32_t b1, uint32_t b2) -> bool {
            if (dr_hi - s.rng_block < X_NEED) {
                refill();
                if (dr_hi - s.rng_block < X_NEED) {
                    s.status = 1;
                    return false;
                }
            }
            // FIFO ring room for this insert's stamp, checked before any state changes
            if (s.next_stamp - s.fifo_head >= d.fifo_cap) {
                drain();  // pending chains write FIFO entries
                while (s.fifo_head < s.next_stamp && d.fifo[s.fifo_head & fmask] < 0) s.fifo_head++;
                if (s.next_stamp - s.fifo_head >= d.fifo_cap) {
                    s.status = 2;
                    return false;
                }
            }
            uint32_t dropped = 0, gc = 0, disp = 0;
            s.writes++;                     // :62
            if (s.live == d.capacity) {     // :64-69 FIFO GC of the oldest entry
                drain();                    // it reads and clears metadata a pending chain writes
                while (d.fifo[s.fifo_head & fmask] < 0) s.fifo_head++;
                const uint32_t f = uint32_t(d.fifo[s.fifo_head & fmask]);
                used_bits[f >> 5] &= ~(1u << (f & 31));  // clear() (:48-54)
                if (lane == 0) {
                    d.fifo[d.stamp[f] & fmask] = -1;
                    d.beta1[f] = 0;
                    d.beta2[f] = 0;
                    d.stamp[f] = 0;
                    touch_store(f, -1);
                }
                s.live--;
                gc = 1;
                __syncwarp();
            }
            const uint64_t stamp = s.next_stamp++;  // :71 (ring room checked above)
            const uint32_t m1 = free_mask(b1);  // :73-84
            const uint32_t m2 = m1 ? 0u : free_mask(b2);
            if (m1 | m2) {
                const uint32_t b = m1 ? b1 : b2;
                const uint32_t f = b * depth + uint32_t(__ffs(int(m1 ? m1 : m2)) - 1);
                used_bits[f >> 5] |= 1u << (f & 31);
                alt_swap(f, b1 ^ b2);
                if (lane == 0) {
                    d.beta1[f] = b1;
                    d.beta2[f] = b2;
                    d.stamp[f] = stamp;
                    d.fifo[stamp & fmask] = int64_t(f);
                    touch_store(f, int64_t(i));
                }
                s.live++;
            } else {
                // :86-125 random-walk eviction, control flow on chip; chain logged
                uint32_t be = uniform(2) == 0 ? b1 : b2;
                uint32_t calt = b1 ^ b2;  // alternate-bucket key of the carried item
                uint32_t h = 0, final_slot = FULLM;
                uint32_t myv = 0;  // lane k < 32 logs chain[k]; longer chains go to chain[]
                for (;; ++h) {
                    const uint64_t dnext = ring[s.rng_block & (X_RING - 1)];  // issued before the test
                    // power-of-two depth: the victim slot is known before the occupancy
                    // test, so its shared-memory alt entry is read alongside it
                    const uint32_t vf_spec = be * depth + (uint32_t(dnext) & (depth - 1));
                    const bool spec = dpow2 && vf_spec < X_SM_SLOTS;
                    const uint32_t va_spec = spec ? alt[vf_spec] : 0u;
                    const uint32_t fm = free_mask(be);
                    if (fm) {
                        final_slot = be * depth + uint32_t(__ffs(int(fm)) - 1);
                        used_bits[final_slot >> 5] |= 1u << (final_slot & 31);
                        alt_swap(final_slot, calt);
                        s.live++;
                        break;
                    }
                    if (h == XPIR_MAX_DISPLACEMENTS_DEV) break;
                    uint32_t vs;
                    if (dpow2) {  // rng.cpp:9-16 without rejection
                        vs = uint32_t(dnext) & (depth - 1);
                        s.rng_block++;
                    } else {
                        vs = uint32_t(uniform(depth));
                    }
                    const uint32_t vf = be * depth + vs;
                    if (h < 32) {
                        if (lane == h) myv = vf;
                    } else {
                        if (h == 32) {  // chain[] is free once warp 1 is done with the last long chain
                            wait_zero(2);
                            chain[lane] = myv;
                        }
                        chain[h] = vf;
                    }
                    uint32_t va;  // the victim's key; the carry takes the slot
                    if (spec) {
                        alt[vf] = uint16_t(calt);
                        va = va_spec;
                    } else {
                        va = alt_swap(vf, calt);
                    }
                    calt = va;
                    be ^= va;  // :118 (beta1 ^ beta2 ^ be is the victim's other bucket)
                }
                disp = final_slot == FULLM ? XPIR_MAX_DISPLACEMENTS_DEV : h;
                dropped = final_slot == FULLM ? 1u : 0u;
                // hand the chain to warp 1, which writes its metadata while this warp goes
                // on (the walk itself reads only on-chip state)
                wait_zero(wslot);
                XRec& r = recs[wslot];
                r.v[lane] = myv;
                if (lane == 0) {
                    r.h = h;
                    r.final_slot = final_slot;
                    r.b1 = b1;
                    r.b2 = b2;
                    r.stamp = stamp;
                    r.i = i;
                    if (h > 32) qflag[2] = 1;
                }
                __syncwarp();
                __threadfence_block();
                if (lane == 0) qflag[wslot] = 1;
                __syncwarp();
                wslot ^= 1;
            }
            if (reports && lane == 0) reinterpret_cast<uint4*>(reports)[i] = make_uint4(1, dropped, gc, disp);
            return true;
        };

        uint64_t c = i0;
        bool stop = false;
        while (c < n && !stop) {
            const uint64_t c0 = c;
            const uint32_t cn = uint32_t((n - c0) < X_CHUNK ? (n - c0) : X_CHUNK);
            for (uint32_t k = lane; k < cn; k += 32) {
                sb1[k] = beta1[c0 + k];
                sb2[k] = beta2[c0 + k];
            }
            __syncwarp();
            const uint64_t ce = c0 + cn;
            while (c < ce) {
                // ---- parallel batch of simple inserts (see k_cuckoo_walk_w) ------
                const uint32_t avail = uint32_t((ce - c) < 32 ? (ce - c) : 32);
                const bool valid = lane < avail;
                const uint32_t b1 = valid ? sb1[c - c0 + lane] : 0u, b2 = valid ? sb2[c - c0 + lane] : 0u;
                const uint32_t m1 = valid ? free_mask(b1) : 0u, m2 = valid ? free_mask(b2) : 0u;
                const bool simple = (m1 | m2) != 0;
                const uint32_t pb = m1 ? b1 : b2, pm = m1 ? m1 : m2;
                if (simple) atomicMin(&htag[pb & (X_HT - 1)], lane);
                __syncwarp();
                const bool conflict = valid && (htag[b1 & (X_HT - 1)] < lane || htag[b2 & (X_HT - 1)] < lane);
                __syncwarp();
                if (simple) htag[pb & (X_HT - 1)] = FULLM;
                const uint64_t room_gc = d.capacity - s.live;
                const uint64_t room_fifo = d.fifo_cap - (s.next_stamp - s.fifo_head);
                const bool halt = !simple || conflict || lane >= room_gc || lane >= room_fifo;
                const uint32_t hm = __ballot_sync(FULLM, halt);
                const uint32_t Lb = hm ? uint32_t(__ffs(int(hm)) - 1) : 32u;
                uint32_t f = 0;
                if (lane < Lb) {
                    const uint64_t i = c + lane;
                    f = pb * depth + uint32_t(__ffs(int(pm)) - 1);
                    const uint64_t stamp = s.next_stamp + lane;
                    atomicOr(&used_bits[f >> 5], 1u << (f & 31));
                    if (f < X_SM_SLOTS) alt[f] = uint16_t(b1 ^ b2);
                    d.beta1[f] = b1;
                    d.beta2[f] = b2;
                    d.stamp[f] = stamp;
                    d.fifo[stamp & fmask] = int64_t(f);
                    touch_store(f, int64_t(i));
                    if (reports) reinterpret_cast<uint4*>(reports)[i] = make_uint4(1, 0, 0, 0);
                }
                // TMEM-resident alt entries of the placed slots, one warp-uniform update each
                uint32_t tmw = __ballot_sync(FULLM, lane < Lb && f >= X_SM_SLOTS);
                while (tmw) {
                    const int src = __ffs(int(tmw)) - 1;
                    tmw &= tmw - 1;
                    const uint32_t ff = __shfl_sync(FULLM, f, src);
                    const uint32_t x = __shfl_sync(FULLM, b1 ^ b2, src);
                    alt_swap(ff, x);
                }
                s.writes += Lb;
                s.live += Lb;
                s.next_stamp += Lb;
                c += Lb;
                __syncwarp();
                if (Lb < 32 && c < ce) {
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
        drain();
        if (lane == 0) qflag[3] = 1;  // done: warp 1 exits
        s.resume_at = c;
        if (lane == 0) *gst = s;
        __threadfence_block();
    } else if (warp == 1) {
        // the resolver: chains in hand-off order
        uint32_t rslot = 0;
        for (;;) {
            uint32_t full;
            while ((full = qflag[rslot]) == 0) {
                if (qflag[3]) {
                    full = qflag[rslot];
                    break;
                }
                __nanosleep(32);
            }
            __syncwarp();
            if (full == 0) break;
            __threadfence_block();
            const XRec& r = recs[rslot];
            const bool lng = r.h > 32;
            resolve_chain(r);
            __syncwarp();
            __threadfence_block();
            if (lane == 0) {
                if (lng) qflag[2] = 0;
                qflag[rslot] = 0;
            }
            __syncwarp();
            rslot ^= 1;
        }
    }
    __syncthreads();
    // occupancy back to the byte map; touched list rebuilt from the marks
    for (uint32_t w = threadIdx.x; w < L.words; w += blockDim.x) {
        const uint32_t v = used_bits[w];
        for (uint32_t k = 0; k < 32 && w * 32 + k < slots; ++k) d.used[w * 32 + k] = (v >> k) & 1u;
    }
    {
        // touched list = slots marked this round, in slot order: each warp owns a
        // contiguous range and walks it 32 slots at a time (coalesced mark loads,
        // ballot + popcount offsets)
        __shared__ uint32_t wcnt[8];
        const uint32_t bid = s.batch_id;
        const uint32_t nwarps = blockDim.x >> 5;
        const uint32_t per = ((slots + nwarps - 1) / nwarps + 31) & ~31u;
        const uint32_t f0 = min(slots, warp * per), f1 = min(slots, f0 + per);
        uint32_t c = 0;
        for (uint32_t f = f0 + lane; f < f1 + lane; f += 32) {
            const bool t = f < f1 && d.touched_mark[f] == bid;
            c += __popc(__ballot_sync(FULLM, t));
        }
        if (lane == 0) wcnt[warp] = c;
        __syncthreads();
        uint32_t o = 0, total = 0;
        for (uint32_t q = 0; q < nwarps; ++q) {
            if (q < warp) o += wcnt[q];
            total += wcnt[q];
        }
        for (uint32_t f = f0 + lane; f < f1 + lane; f += 32) {
            const bool t = f < f1 && d.touched_mark[f] == bid;
            const uint32_t m = __ballot_sync(FULLM, t);
            if (t) d.touched[o + __popc(m & ((1u << lane) - 1u))] = f;
            o += __popc(m);
        }
        if (threadIdx.x == 0) gst->n_touched = total;
    }
    if (use_tm) {
        asm volatile("tcgen05.fence::before_thread_sync;\n");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
    }
}

cudaError_t launch_cuckoo_walk_x(const CuckooDev& d, CuckooState* st, const uint32_t* beta1, const uint32_t* beta2,
                                 uint64_t i0, uint64_t n, uint32_t* reports, cudaStream_t s) {
    const XLayout L(uint32_t(uint64_t(d.buckets) * d.depth));
    auto k = d.depth == 4 ? k_cuckoo_walk_x<4> : k_cuckoo_walk_x<0>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L.total));
    if (e != cudaSuccess) return e;
    k<<<1, 256, L.total, s>>>(d, st, beta1, beta2, i0, n, reports);
    return cudaGetLastError();
}

}  // namespace xpir
