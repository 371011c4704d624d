// K6a: exact parallel placement for the eviction-free prefix of a write round.
//
// cuckoo::Table::insert (cuckoo.cpp:56-126) is sequential: insert i takes the
// lowest free slot of beta1, else of beta2, else starts an eviction walk. As
// long as no eviction and no FIFO GC happens, slots are only ever added, so the
// outcome of insert i depends only on how many EARLIER claims each of its
// buckets received: bucket b admits exactly its first free0(b) claims (in
// insert order) and the k-th admitted claim takes b's k-th free slot.
//
// Each insert claims beta1; an insert whose beta1 claim fails also claims
// beta2. The claim set is solved by Jacobi iteration: sort claims by
// (bucket, insert, which) with CUB, rank each claim within its bucket
// (binary search for the bucket's first claim), update the outcomes, repeat.
// The sequential result is the unique fixed point (by induction on the insert
// index), so once no outcome changes below the first insert that needs an
// eviction, the prefix before it is exactly what the sequential code produces.
// That prefix is applied in parallel (same metadata, FIFO stamps and payload
// origins as the walk writes); k_cuckoo_walk continues from the first eviction.
#include <cuda_runtime.h>

#include <cub/cub.cuh>
#include <cstdint>

#include "scan.cuh"

namespace xpir {

namespace {

__global__ void k_par_keys(uint64_t n, const uint32_t* __restrict__ b1, const uint32_t* __restrict__ b2,
                           const uint8_t* __restrict__ outcome, unsigned long long* __restrict__ keys) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    keys[2 * i] = (unsigned long long)b1[i] << 32 | (2 * i);
    keys[2 * i + 1] = outcome[i] >= 2 ? ((unsigned long long)b2[i] << 32 | (2 * i + 1)) : ~0ull;
}

__device__ __forceinline__ uint32_t first_of_bucket(const unsigned long long* __restrict__ k, uint64_t p,
                                                    uint32_t b) {
    // smallest q <= p with (k[q] >> 32) == b (keys sorted ascending)
    uint64_t lo = 0, hi = p;
    const unsigned long long target = (unsigned long long)b << 32;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (k[mid] < target) lo = mid + 1;
        else hi = mid;
    }
    return uint32_t(p - lo);
}

__device__ __forceinline__ uint32_t free_slots(const uint8_t* __restrict__ used, uint32_t b, uint32_t depth) {
    uint32_t f = 0;
    for (uint32_t s = 0; s < depth; ++s) f += used[uint64_t(b) * depth + s] ? 0u : 1u;
    return f;
}

__global__ void k_par_rank(const unsigned long long* __restrict__ k, uint64_t m, const uint8_t* __restrict__ used,
                           uint32_t depth, uint8_t* __restrict__ succ) {
    const uint64_t p = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= m) return;
    const unsigned long long key = k[p];
    if (key == ~0ull) return;
    const uint32_t b = uint32_t(key >> 32), c = uint32_t(key);
    succ[c] = first_of_bucket(k, p, b) < free_slots(used, b, depth) ? 1 : 0;
}

// flags[0] = min insert whose outcome changed, flags[1] = min insert needing an eviction
__global__ void k_par_update(uint64_t n, uint8_t* __restrict__ outcome, const uint8_t* __restrict__ succ,
                             unsigned long long* __restrict__ flags) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint8_t o = outcome[i];
    const uint8_t nw = succ[2 * i] ? 1 : (o >= 2 ? (succ[2 * i + 1] ? 2 : 3) : 2);
    if (nw != o) {
        outcome[i] = nw;
        atomicMin(&flags[0], (unsigned long long)i);
    }
    if (nw == 3) atomicMin(&flags[1], (unsigned long long)i);
}

// placing claim -> flat slot (from the pre-round occupancy)
__global__ void k_par_slot(const unsigned long long* __restrict__ k, uint64_t m, const uint8_t* __restrict__ used,
                           uint32_t depth, const uint8_t* __restrict__ outcome, uint64_t limit,
                           uint32_t* __restrict__ slot_of) {
    const uint64_t p = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= m) return;
    const unsigned long long key = k[p];
    if (key == ~0ull) return;
    const uint32_t b = uint32_t(key >> 32), c = uint32_t(key);
    const uint32_t i = c >> 1, which = c & 1;
    if (i >= limit || outcome[i] != which + 1) return;
    uint32_t r = first_of_bucket(k, p, b);
    for (uint32_t s = 0; s < depth; ++s) {
        if (used[uint64_t(b) * depth + s]) continue;
        if (r == 0) {
            slot_of[i] = b * depth + s;
            return;
        }
        --r;
    }
}

__global__ void k_par_write(CuckooDev d, uint64_t limit, const uint32_t* __restrict__ b1,
                            const uint32_t* __restrict__ b2, const uint32_t* __restrict__ slot_of,
                            uint64_t next_stamp, uint32_t batch_id, uint32_t touched0,
                            uint32_t* __restrict__ reports) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= limit) return;
    const uint32_t f = slot_of[i];
    const uint64_t stamp = next_stamp + i;  // cuckoo.cpp:71, one stamp per insert
    d.used[f] = 1;                           // cuckoo.cpp:37-46
    d.beta1[f] = b1[i];
    d.beta2[f] = b2[i];
    d.stamp[f] = stamp;
    d.fifo[stamp & (d.fifo_cap - 1)] = int64_t(f);
    d.origin[f] = int64_t(i);
    d.touched_mark[f] = batch_id;
    d.touched[touched0 + i] = f;
    if (reports) reinterpret_cast<uint4*>(reports)[i] = make_uint4(1, 0, 0, 0);
}

}  // namespace

// Runs on the first `n` inserts of a batch whose walk state is `h` (host copy,
// batch_id set, n_touched == 0, no GC possible within n). Returns the length k
// of the eviction-free prefix it applied (0 if it declined) and advances h.
// Keys are (bucket << 32 | 2*insert + which), written in ascending insert order,
// and CUB's radix sort is stable: sorting the bucket field alone (bits 32 ..
// end_bit) yields the (bucket, insert, which) order in ceil(log2(buckets+1)) / 8
// passes instead of 6. The field is one bit wider than the largest bucket so the
// ~0 "no claim" keys sort after every real bucket.
static int sort_end_bit(uint32_t buckets) {
    int end_bit = 32;
    while (end_bit < 64 && (uint64_t(1) << (end_bit - 32)) <= buckets) ++end_bit;
    return end_bit;
}

cudaError_t cuckoo_reserve(CuckooParScratch& sc, uint64_t n, uint32_t buckets, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const uint64_t m = 2 * n;
    cudaError_t e = cudaSuccess;
    auto grow = [&](void** p, size_t bytes, size_t& cap) {
        if (e != cudaSuccess || bytes <= cap) return;
        if (*p) cudaFree(*p);
        *p = nullptr;
        cap = 0;
        e = cudaMalloc(p, bytes);
        if (e == cudaSuccess) cap = bytes;
    };
    grow(&sc.keys_a, m * 8, sc.keys_a_cap);
    grow(&sc.keys_b, m * 8, sc.keys_b_cap);
    grow(&sc.outcome, n, sc.outcome_cap);
    grow(&sc.succ, m, sc.succ_cap);
    grow(&sc.slot_of, n * 4, sc.slot_cap);
    grow(&sc.flags, 16, sc.flags_cap);
    if (e != cudaSuccess) return e;
    size_t tmp = 0;
    e = cub::DeviceRadixSort::SortKeys(nullptr, tmp, static_cast<unsigned long long*>(sc.keys_a),
                                       static_cast<unsigned long long*>(sc.keys_b), int(m), 32,
                                       sort_end_bit(buckets), s);
    if (e != cudaSuccess) return e;
    grow(&sc.cub_tmp, tmp, sc.cub_cap);
    return e;
}

cudaError_t cuckoo_parallel_prefix(const CuckooDev& d, CuckooState& h, const uint32_t* b1, const uint32_t* b2,
                                   uint64_t n, uint32_t* reports, CuckooParScratch& sc, uint64_t* applied,
                                   cudaStream_t s) {
    *applied = 0;
    if (n == 0) return cudaSuccess;
    const uint64_t m = 2 * n;
    cudaError_t e = cuckoo_reserve(sc, n, d.buckets, s);
    if (e != cudaSuccess) return e;
    const int end_bit = sort_end_bit(d.buckets);
    auto* keys_in = static_cast<unsigned long long*>(sc.keys_a);
    auto* keys = static_cast<unsigned long long*>(sc.keys_b);
    auto* outcome = static_cast<uint8_t*>(sc.outcome);
    auto* succ = static_cast<uint8_t*>(sc.succ);
    auto* flags = static_cast<unsigned long long*>(sc.flags);
    const uint32_t gn = uint32_t((n + 255) / 256), gm = uint32_t((m + 255) / 256);
    if ((e = cudaMemsetAsync(outcome, 1, n, s)) != cudaSuccess) return e;
    uint64_t k = 0;
    bool converged = false;
    // Iterations run in pairs between host checks: once the fixed point is reached
    // a further iteration changes nothing, so the pair's last flags decide.
    for (int it = 0; it < 48; it += 2) {
        for (int rep = 0; rep < 2; ++rep) {
            k_par_keys<<<gn, 256, 0, s>>>(n, b1, b2, outcome, keys_in);
            size_t tb = sc.cub_cap;
            e = cub::DeviceRadixSort::SortKeys(sc.cub_tmp, tb, keys_in, keys, int(m), 32, end_bit, s);
            if (e != cudaSuccess) return e;
            k_par_rank<<<gm, 256, 0, s>>>(keys, m, d.used, d.depth, succ);
            if ((e = cudaMemsetAsync(flags, 0xff, 16, s)) != cudaSuccess) return e;
            k_par_update<<<gn, 256, 0, s>>>(n, outcome, succ, flags);
        }
        unsigned long long f[2];
        if ((e = cudaMemcpyAsync(f, flags, 16, cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
        if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
        count_launches(8);
        const uint64_t first_evict = f[1] == ~0ull ? n : f[1];
        const uint64_t first_change = f[0] == ~0ull ? n : f[0];
        if (first_change >= first_evict) {
            k = first_evict;
            converged = true;
            break;
        }
    }
    if (!converged || k == 0) return cudaGetLastError();
    k_par_slot<<<gm, 256, 0, s>>>(keys, m, d.used, d.depth, outcome, k, static_cast<uint32_t*>(sc.slot_of));
    k_par_write<<<uint32_t((k + 255) / 256), 256, 0, s>>>(d, k, b1, b2, static_cast<uint32_t*>(sc.slot_of),
                                                         h.next_stamp, h.batch_id, h.n_touched, reports);
    count_launches(2);
    h.writes += k;
    h.live += k;
    h.next_stamp += k;
    h.n_touched += uint32_t(k);
    *applied = k;
    return cudaGetLastError();
}

}  // namespace xpir
