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
// beta2. Both potential claims of every insert are grouped by bucket ONCE
// (count, scan, scatter — order inside a group is irrelevant); the claim set is
// then solved by Jacobi iteration inside one cooperative kernel: each active
// claim counts the active claims with a smaller claim id in its bucket's group,
// grid barrier, each insert updates its outcome, grid barrier, convergence test
// on device — one launch and one 24-byte read back per round, no host round
// trip per iteration.
// The sequential result is the unique fixed point (by induction on the insert
// index), so once no outcome changes below the first insert that needs an
// eviction, the prefix before it is exactly what the sequential code produces.
// That prefix is applied in parallel (same metadata, FIFO stamps and payload
// origins as the walk writes); k_cuckoo_walk continues from the first eviction.
#include <cuda_runtime.h>

#include <cooperative_groups.h>
#include <cstdint>

#include "scan.cuh"

namespace xpir {

namespace {


// flags (zero-initialised once at allocation; the kernel leaves its working
// slots reset for the next launch): [0..1] min insert whose outcome changed
// (iteration parity), [2..3] min insert needing an eviction (parity), [5] abort
// (a bucket group too long to scan: decline, the walk places the round), [6]
// first insert with a bucket out of range (cuckoo.cpp:57-58); results for the
// host: [8] k, [9] first bad insert (n when none).
constexpr int PAR_SOLVE_NT = 512;
constexpr uint32_t PAR_MAX_SCAN = 4096;
constexpr uint32_t PAR_MAX_BLOCKS = 2048;
constexpr unsigned long long NONE = ~0ull;

__device__ __forceinline__ uint32_t claim_bucket(const uint32_t* __restrict__ b1, const uint32_t* __restrict__ b2,
                                                 uint32_t c) {
    return (c & 1) ? b2[c >> 1] : b1[c >> 1];
}

// Exclusive scan of one value per thread across the block; *total = block sum.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* total) {
    __shared__ uint32_t warp_sum[PAR_SOLVE_NT / 32];
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= uint32_t(off)) x += y;
    }
    if (lane == 31) warp_sum[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t t = lane < PAR_SOLVE_NT / 32 ? warp_sum[lane] : 0;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, t, off);
            if (lane >= uint32_t(off)) t += y;
        }
        if (lane < PAR_SOLVE_NT / 32) warp_sum[lane] = t;  // inclusive
    }
    __syncthreads();
    const uint32_t before = (w ? warp_sum[w - 1] : 0) + x - v;
    *total = warp_sum[PAR_SOLVE_NT / 32 - 1];
    __syncthreads();  // warp_sum is reused by the next call
    return before;
}

// One cooperative grid for the whole eviction-free prefix (7 grid barriers at two
// Jacobi iterations):
//  P0  range check of every beta, per-bucket counts cnt[] of every potential
//      claim (beta1 and beta2 of every insert), outcome = "claims beta1";
//  P1  each block scans its bucket chunk: loc[b] = claims of the chunk's buckets
//      before b, chunk_sum[block];
//  P2  every block prefix-sums chunk_sum in shared memory (chunk offsets), and
//      the claims are grouped by bucket: group of b = [loc[b] + off(chunk(b)), +cnt[b]);
//  Jacobi iterations: A — every active claim succeeds iff fewer than the
//      bucket's free slots of the active claims in its group have a smaller claim
//      id (group order is irrelevant); a succeeding claim also records its slot
//      (the rank-th free slot of the pre-round bucket); B — outcome update;
//      convergence tested on device;
//  apply — the placing claims below the first eviction write their slots
//      (cuckoo.cpp:37-46, one stamp per insert, :71); cnt[] / cur[] are cleared for
//      the next launch.
__global__ void __launch_bounds__(PAR_SOLVE_NT)
k_par_solve(CuckooDev d, CuckooState* st, uint64_t n, const uint32_t* __restrict__ b1,
            const uint32_t* __restrict__ b2, uint32_t* cnt, uint32_t* loc, uint32_t* cur, uint32_t* chunk_sum,
            uint32_t* grouped, uint8_t* outcome, uint8_t* succ, uint32_t* slot_of,
            unsigned long long* flags, uint32_t* __restrict__ reports, int max_iters) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ uint32_t off[PAR_MAX_BLOCKS + 1];
    const uint64_t tid = grid.thread_rank(), nthr = grid.size();
    volatile unsigned long long* vf = flags;
    const uint32_t NB = d.buckets;
    // the batch's starting state (read by every thread before thread 0 changes it)
    const uint64_t live0 = st->live, next_stamp = st->next_stamp, head = st->fifo_head;
    const uint32_t batch_id = st->batch_id + 1;
    // no FIFO GC within the prefix, and every new stamp must fit the FIFO ring
    const uint64_t span = next_stamp - head;
    const uint64_t ring_room = d.fifo_cap > span ? d.fifo_cap - span : 0;
    uint64_t room = d.capacity > live0 ? d.capacity - live0 : 0;
    if (room > ring_room) room = ring_room;
    // P0 (cnt and cur are all zero on entry)
    for (uint64_t i = tid; i < n; i += nthr) {
        const uint32_t x1 = b1[i], x2 = b2[i];
        if (x1 >= NB || x2 >= NB) {
            atomicMin(flags + 6, (unsigned long long)i);
            continue;
        }
        outcome[i] = 1;  // everyone claims beta1 first
        atomicAdd(cnt + x1, 1u);
        atomicAdd(cnt + x2, 1u);
    }
    grid.sync();
    const unsigned long long fb = vf[6];
    const uint64_t n_ok = fb == NONE ? n : fb;
    const uint64_t ne = n_ok < room ? n_ok : room;
    // P1: chunk scans
    const uint32_t nblk = gridDim.x, per = (NB + nblk - 1) / nblk;
    {
        const uint32_t c0 = min(NB, blockIdx.x * per), c1 = min(NB, c0 + per);
        const uint32_t ipt = (per + PAR_SOLVE_NT - 1) / PAR_SOLVE_NT;  // buckets per thread
        const uint32_t t0 = min(c1, c0 + threadIdx.x * ipt), t1 = min(c1, t0 + ipt);
        uint32_t v = 0;
        for (uint32_t b = t0; b < t1; ++b) v += __ldcg(cnt + b);
        uint32_t tot;
        uint32_t run = block_exclusive_scan(v, &tot);
        for (uint32_t b = t0; b < t1; ++b) {
            __stcg(loc + b, run);
            run += __ldcg(cnt + b);
        }
        if (threadIdx.x == 0) __stcg(chunk_sum + blockIdx.x, tot);
    }
    grid.sync();
    // P2: chunk offsets in shared memory (every block), then the grouping
    {
        const uint32_t ipt = (nblk + PAR_SOLVE_NT - 1) / PAR_SOLVE_NT;
        const uint32_t t0 = min(nblk, threadIdx.x * ipt), t1 = min(nblk, t0 + ipt);
        uint32_t v = 0;
        for (uint32_t k = t0; k < t1; ++k) v += __ldcg(chunk_sum + k);
        uint32_t tot;
        uint32_t run = block_exclusive_scan(v, &tot);
        for (uint32_t k = t0; k < t1; ++k) {
            off[k] = run;
            run += __ldcg(chunk_sum + k);
        }
        if (threadIdx.x == 0) off[nblk] = tot;
        __syncthreads();
    }
    // every insert with both betas in range, as counted in P0; claims of inserts
    // >= ne stay in their groups but never act (a claim only counts claims with
    // smaller ids, i.e. of earlier inserts)
    for (uint64_t c = tid; c < 2 * n; c += nthr) {
        const uint32_t x1 = b1[c >> 1], x2 = b2[c >> 1];
        if (x1 >= NB || x2 >= NB) continue;
        const uint32_t b = (c & 1) ? x2 : x1;
        grouped[__ldcg(loc + b) + off[b / per] + atomicAdd(cur + b, 1u)] = uint32_t(c);
    }
    grid.sync();
    const uint32_t G = off[nblk];  // claims grouped
    uint64_t k = 0;
    bool conv = false;
    for (int it = 0; it < max_iters; ++it) {
        const int par = it & 1;
        if (tid == 0) {  // this parity was last read two iterations ago
            vf[par] = NONE;
            vf[2 + par] = NONE;
        }
        // A: every active claim counts the active claims with a smaller id in its
        // bucket's group (group order is irrelevant)
        for (uint64_t p = tid; p < G; p += nthr) {
            const uint32_t c = grouped[p];
            if ((c >> 1) >= ne) continue;
            if ((c & 1) && __ldcg(outcome + (c >> 1)) < 2) continue;  // beta2 claim not made
            const uint32_t b = claim_bucket(b1, b2, c);
            const uint8_t* u = d.used + uint64_t(b) * d.depth;
            uint32_t fr = 0;
            for (uint32_t sl = 0; sl < d.depth; ++sl) fr += u[sl] ? 0u : 1u;
            const uint32_t g0 = loc[b] + off[b / per], g1 = g0 + cnt[b];
            uint32_t r = 0;
            if (g1 - g0 > PAR_MAX_SCAN) {
                vf[5] = 1;  // decline: the walk places the round
            } else {
                for (uint32_t q = g0; q < g1; ++q) {
                    const uint32_t cq = grouped[q];
                    if (cq < c && (!(cq & 1) || __ldcg(outcome + (cq >> 1)) >= 2)) ++r;
                }
            }
            const bool ok = r < fr;
            __stcg(succ + c, uint8_t(ok ? 1 : 0));
            if (ok) {  // the r-th free slot of the pre-round bucket (cuckoo.cpp:31-35 order)
                uint32_t sl = 0;
                for (uint32_t left = r;; ++sl)
                    if (!u[sl] && left-- == 0) break;
                __stcg(slot_of + c, b * d.depth + sl);
            }
        }
        grid.sync();
        // B: outcome update (1 = placed in beta1, 2 = claims / placed in beta2, 3 = eviction)
        for (uint64_t i = tid; i < ne; i += nthr) {
            const uint8_t o = __ldcg(outcome + i);
            const uint8_t nw = __ldcg(succ + 2 * i) ? 1 : (o >= 2 ? (__ldcg(succ + 2 * i + 1) ? 2 : 3) : 2);
            if (nw != o) {
                __stcg(outcome + i, nw);
                atomicMin(flags + par, (unsigned long long)i);
            }
            if (nw == 3) atomicMin(flags + 2 + par, (unsigned long long)i);
        }
        grid.sync();
        const bool abort = vf[5] != 0;
        const unsigned long long fc = vf[par], fe = vf[2 + par];
        const uint64_t first_evict = fe == NONE ? ne : fe, first_change = fc == NONE ? ne : fc;
        if (abort) break;
        if (first_change >= first_evict) {
            k = first_evict;
            conv = true;
            break;
        }
    }
    if (!conv) k = 0;
    // apply; every phase that read `used` ended at the last barrier
    for (uint64_t i = tid; i < k; i += nthr) {  // cuckoo.cpp:37-46; one stamp per insert (:71)
        const uint32_t f = __ldcg(slot_of + 2 * i + (__ldcg(outcome + i) - 1));
        const uint64_t stamp = next_stamp + i;
        d.used[f] = 1;
        d.beta1[f] = b1[i];
        d.beta2[f] = b2[i];
        d.stamp[f] = stamp;
        d.fifo[stamp & (d.fifo_cap - 1)] = int64_t(f);
        d.origin[f] = int64_t(i);
        d.touched_mark[f] = batch_id;
        d.touched[i] = f;
        if (reports) reinterpret_cast<uint4*>(reports)[i] = make_uint4(1, 0, 0, 0);
    }
    for (uint64_t b = tid; b < NB; b += nthr) {  // counters zero for the next launch
        __stcg(cnt + b, 0u);
        __stcg(cur + b, 0u);
    }
    if (tid == 0) {
        vf[8] = k;
        vf[9] = n_ok;
        vf[5] = 0;
        vf[6] = NONE;
        CuckooState x = *st;
        x.batch_id = batch_id;
        x.writes += k;
        x.live += k;
        x.next_stamp += k;
        x.n_touched = uint32_t(k);
        x.resume_at = k;
        x.limit = n_ok;
        x.status = 0;
        x.walked = 0;
        *st = x;
    }
}

}  // namespace

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
    // per bucket: counts, chunk-local starts, cursors (counts and cursors zero between
    // launches); chunk sums
    const size_t kcap0 = sc.keys_a_cap;
    grow(&sc.keys_a, (3 * uint64_t(buckets) + PAR_MAX_BLOCKS) * 4, sc.keys_a_cap);
    if (e == cudaSuccess && sc.keys_a_cap != kcap0) e = cudaMemsetAsync(sc.keys_a, 0, sc.keys_a_cap, s);
    grow(&sc.keys_b, m * 4, sc.keys_b_cap);                            // claims grouped by bucket
    grow(&sc.outcome, n, sc.outcome_cap);
    grow(&sc.succ, m, sc.succ_cap);
    grow(&sc.slot_of, m * 4, sc.slot_cap);  // per claim
    if (e == cudaSuccess && !sc.flags) {
        grow(&sc.flags, 128, sc.flags_cap);
        if (e == cudaSuccess) e = cudaMemsetAsync(sc.flags, 0xff, 128, s);  // NONE everywhere
        if (e == cudaSuccess) e = cudaMemsetAsync(static_cast<unsigned long long*>(sc.flags) + 5, 0, 8, s);
    }
    return e;
}

cudaError_t cuckoo_parallel_prefix(const CuckooDev& d, CuckooState* st, const uint32_t* b1, const uint32_t* b2,
                                   uint64_t n, uint32_t* reports, CuckooParScratch& sc, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    cudaError_t e = cuckoo_reserve(sc, n, d.buckets, s);
    if (e != cudaSuccess) return e;
    static int per_sm = 0, sms = 0;
    if (!per_sm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_par_solve, PAR_SOLVE_NT, 0);
        if (per_sm < 1) per_sm = 1;
    }
    const uint64_t want = (2 * n + PAR_SOLVE_NT - 1) / PAR_SOLVE_NT;
    const uint64_t cap = uint64_t(per_sm) * sms;
    uint32_t blocks = uint32_t(want < 1 ? 1 : want > cap ? cap : want);
    if (blocks > PAR_MAX_BLOCKS) blocks = PAR_MAX_BLOCKS;  // chunk_sum entries
    CuckooDev dd = d;
    uint64_t nn = n;
    auto* cnt = static_cast<uint32_t*>(sc.keys_a);
    uint32_t* loc = cnt + d.buckets;
    uint32_t* cur = loc + d.buckets;
    uint32_t* chunk_sum = cur + d.buckets;
    auto* grouped = static_cast<uint32_t*>(sc.keys_b);
    auto* outcome = static_cast<uint8_t*>(sc.outcome);
    auto* succ = static_cast<uint8_t*>(sc.succ);
    auto* slot_of = static_cast<uint32_t*>(sc.slot_of);
    auto* flags = static_cast<unsigned long long*>(sc.flags);
    int iters = 64;
    void* args[] = {&dd, &st, &nn, (void*)&b1, (void*)&b2, &cnt, &loc, &cur, &chunk_sum, &grouped, &outcome,
                    &succ, &slot_of, &flags, &reports, &iters};
    e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_par_solve), dim3(blocks), dim3(PAR_SOLVE_NT), args, 0,
                                    s);
    if (e != cudaSuccess) return e;
    count_launches(1);
    return cudaSuccess;
}

}  // namespace xpir
