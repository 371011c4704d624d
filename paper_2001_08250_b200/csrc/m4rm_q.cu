// K1 (B >= 2048): M4RM byte tables over 32-byte columns, four tables
// interleaved per bank row, accumulators entirely in Tensor Memory.
//
// Same math as k_scan_m4rm / k_scan_m4rm_tmem: query byte g of request r
// selects buckets 8g..8g+7 (pir.hpp:25); T_g[x] = XOR_{i in x} bucket_{8g+i};
// the answer slice is the XOR over g of T_g[q_r[g]] (bit-exact
// pir::answer_batch, pir.cpp:41-52).
//
// What changes against k_scan_m4rm_tmem (128-byte columns, Rc = 2048):
//  * A "set" is four consecutive groups g = 4j..4j+3. Their four tables share
//    one 32 KiB buffer: row x of table t sits at x*128 + 32t, so each table row
//    is 32 bytes (one column tile) and the four tables of a row fill one
//    128-byte bank line.
//  * One lane owns one request and its full 32-byte slice (two 16-byte halves).
//    In step kk of a set, lane i of a quarter-warp reads table
//    t = ((i>>1) + kk) & 3, half (i&1) first: the eight lanes of a quarter-warp
//    always hit eight distinct 16-byte bank groups, so every LDS.128 is a
//    single conflict-free wavefront per quarter-warp, for any query bytes.
//  * Accumulators: 32 bytes x 16 requests per thread = all 256 KiB of TMEM
//    (tcgen05.ld/st .32x32b.x8), read-modify-written once per set (4 groups),
//    so TMEM traffic is half the lookup bytes. Rc = 8192 requests per tile.
//  * Shared-memory wavefronts per set (per SM, Rc = 8192): 8192 lookups,
//    320 table build (4 tables x 256 rows x 32 B + bucket reads), 256 query
//    index loads, 8 bucket fills: lookups are 93% of the pipe (the 128-byte
//    column kernel: 82%), because the table build is amortised over 4x more
//    requests and each index byte now serves 32 bytes of lookup instead of 16.
//    Measured (ncu, 1 GiB, B = 8192): LSU data pipe 95% busy, 0 load bank
//    conflicts, lookups 89% of the shared wavefronts; 0.87 of the LDS.128 peak.
//  * Query index bytes come in a set-interleaved layout (one 32-bit word of the
//    set's four group bytes per request, written so by k_expand_T /
//    k_transpose_q) and are read straight from L2 into registers one set ahead
//    (LDG.128 = 4 requests per lane), so they never pass through shared memory;
//    bucket slices are staged by cp.async (zero-fill past the shard).
//
// TMEM map (one CTA per SM): warp w uses lanes 32*(w%4)..+31 and columns
// 128*(w/4) + 8*s for its request slot s < 4*NQ.
#include <cuda_runtime.h>

#include <cstdint>

#include "ptx.cuh"
#include "scan.cuh"

namespace xpir {

using namespace ptx;

namespace {

constexpr int Q_NT = 512;
constexpr int Q_TAB = 256 * 128;  // one set of four interleaved tables
constexpr int Q_NST = 4;          // staging ring depth (sets)

template <int NQ>
struct QCfg {
    static constexpr int RC = Q_NT * 4 * NQ;  // requests per tile
    static constexpr int STG = 1024;          // 32 buckets x 32 B per staged set
    static constexpr int OFF_STG = 2 * Q_TAB;
    static constexpr int OFF_ADDR = OFF_STG + Q_NST * STG;
    static constexpr int SMEM = OFF_ADDR + 16;
    static constexpr int TCOLS = 128 * NQ;  // TMEM columns (power of two >= 32)
    static_assert(SMEM <= 232448, "exceeds the 227 KB opt-in shared memory per CTA");
};

__device__ __forceinline__ void tm_ld8(uint32_t a, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                   "=r"(v[7])
                 : "r"(a));
}
__device__ __forceinline__ void tm_st8(uint32_t a, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(a),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
}
// wait::ld with the destination registers as in/out operands so no use of them
// is scheduled before the wait.
__device__ __forceinline__ void tm_wait_ld8(uint32_t (&v)[8]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;\n"
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]),
                   "+r"(v[7])
                 :
                 : "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
// query words: read once per CTA, reused through L2 by the other column tiles
// (evict_last: the ~128 CTAs of a segment re-read each set from L2, not DRAM)
__device__ __forceinline__ uint4 ldg_q(const uint8_t* p, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;\n"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
    return pol;
}

}  // namespace

template <int NQ>
__global__ void __launch_bounds__(Q_NT, 1)
k_scan_m4rm_q(const uint8_t* __restrict__ db, uint32_t nb, uint32_t S, const uint8_t* __restrict__ qT,
              uint64_t qstride, uint32_t B, uint8_t* __restrict__ out, uint32_t n_ctiles, uint32_t n_sets,
              uint32_t n_seg, PeerOut peers) {
    using C = QCfg<NQ>;
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sbase = smem_u32(smem);
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int i8 = lane & 7, lp = i8 >> 1;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                         sbase + C::OFF_ADDR),
                     "n"(C::TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tbase = *reinterpret_cast<const uint32_t*>(smem + C::OFF_ADDR);
    const uint32_t tcol = tbase + (uint32_t((warp & 3) * 32) << 16) + uint32_t(warp >> 2) * (32 * NQ);

    // lookup constants: step kk reads table (lp + kk) & 3, own half first; its index
    // is byte t of the request's set word (PRMT selector 0x4440 | t)
    uint32_t toff[4], bsel[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
        const uint32_t t = uint32_t(lp + kk) & 3u;
        toff[kk] = 32 * t + 16 * uint32_t(i8 & 1);
        bsel[kk] = 0x4440u | t;
    }
    const uint32_t dhalf = (i8 & 1) ? 0xfffffff0u : 16u;  // address of the other half: +16 / -16
    // build constants: lane -> (table bt, 32-bit word bw); warp -> high nibble of the row
    const int bt = lane >> 3, bw = lane & 7;
    const uint32_t hm0 = 0u - (warp & 1u), hm1 = 0u - ((warp >> 1) & 1u), hm2 = 0u - ((warp >> 2) & 1u);

    const uint32_t n_rtiles = (B + C::RC - 1) / C::RC;
    const uint64_t units = uint64_t(n_ctiles) * n_rtiles * n_seg;
    // Staging sequence number of a set over the CTA's lifetime: stage buffer
    // seq % Q_NST, table buffer seq & 1.
    uint32_t seq0 = 0;

    for (uint64_t v = blockIdx.x; v < units; v += gridDim.x) {
        const uint32_t c = uint32_t(v % n_ctiles);
        const uint32_t rt = uint32_t((v / n_ctiles) % n_rtiles);
        const uint32_t sg = uint32_t(v / (uint64_t(n_ctiles) * n_rtiles));
        const uint32_t s0 = uint32_t(uint64_t(n_sets) * sg / n_seg);
        const uint32_t s1 = uint32_t(uint64_t(n_sets) * (sg + 1) / n_seg);
        if (s0 >= s1) continue;
        const uint32_t r_base = rt * C::RC;

        // zero this unit's accumulators
        {
            uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
            for (int s = 0; s < 4 * NQ; ++s) tm_st8(tcol + 8 * s, z);
            tm_wait_st();
        }

        // The bucket slices of column tile c for set j (laid out [i][t][32 B]) are
        // staged by cp.async with zero-fill past the shard. The query words of a set
        // (set-interleaved layout: one 32-bit word of four group bytes per request)
        // are read straight from L2 into registers, one set ahead.
        auto stage = [&](uint32_t j, uint32_t sq) {
            const int buf = int(sq % Q_NST);
            const uint32_t dst = sbase + C::OFF_STG + buf * C::STG;
            if (tid < 64) {
                const uint32_t i = tid >> 3, t = (tid >> 1) & 3, part = tid & 1;
                const uint32_t bucket = (j * 4 + t) * 8 + i;
                const bool ok = bucket < nb;
                const uint8_t* src = db + (ok ? uint64_t(bucket) * S : 0) + uint64_t(c) * 32 + part * 16;
                cp_async16(dst + tid * 16, src, ok ? 16u : 0u);
            }
        };
        const uint64_t qpol = l2_evict_last_policy();
        auto load_q = [&](uint32_t j, uint4 (&w)[NQ]) {
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const uint32_t r4 = r_base + 4 * uint32_t(q * Q_NT + tid);
                w[q] = r4 < qstride ? ldg_q(qT + uint64_t(j) * 4 * qstride + uint64_t(r4) * 4, qpol) : make_uint4(0, 0, 0, 0);
            }
        };
        // Warps 0-7 build (warp w: the rows with high nibble w, then w + 8 — the same
        // 8 bucket words serve both), so the bucket words are read by 8 warps, not 16.
        auto build = [&](int buf, int tb) {
            if (warp >= 8) return;
            const uint32_t src = sbase + C::OFF_STG + buf * C::STG + bt * 32 + bw * 4;
            uint32_t b[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) b[i] = lds32(src + i * 128);
            uint32_t h = (b[4] & hm0) ^ (b[5] & hm1) ^ (b[6] & hm2);
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const uint32_t row0 = sbase + tb * Q_TAB + uint32_t((warp + 8 * half) << 4) * 128 + bt * 32 + bw * 4;
                uint32_t x = half ? h ^ b[7] : h;
                sts32(row0, x);
#pragma unroll
                for (int m = 1; m < 16; ++m) {
                    x ^= b[(m & 1) ? 0 : (m & 2) ? 1 : (m & 4) ? 2 : 3];  // ctz(m)
                    sts32(row0 + uint32_t(m ^ (m >> 1)) * 128, x);
                }
            }
        };
        auto lookups = [&](const uint4 (&wq)[NQ], int tb) {
            const uint32_t tab = sbase + tb * Q_TAB;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const uint32_t wk[4] = {wq[q].x, wq[q].y, wq[q].z, wq[q].w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t ta = tcol + 8 * (4 * q + k);
                    uint32_t m[8];
                    tm_ld8(ta, m);
                    uint4 v0[4], v1[4];
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint32_t a0 = tab + toff[kk] + __byte_perm(wk[k], 0, bsel[kk]) * 128;
                        v0[kk] = lds128(a0);
                        v1[kk] = lds128(a0 + dhalf);
                    }
                    tm_wait_ld8(m);
                    m[0] ^= (v0[0].x ^ v0[1].x) ^ (v0[2].x ^ v0[3].x);
                    m[1] ^= (v0[0].y ^ v0[1].y) ^ (v0[2].y ^ v0[3].y);
                    m[2] ^= (v0[0].z ^ v0[1].z) ^ (v0[2].z ^ v0[3].z);
                    m[3] ^= (v0[0].w ^ v0[1].w) ^ (v0[2].w ^ v0[3].w);
                    m[4] ^= (v1[0].x ^ v1[1].x) ^ (v1[2].x ^ v1[3].x);
                    m[5] ^= (v1[0].y ^ v1[1].y) ^ (v1[2].y ^ v1[3].y);
                    m[6] ^= (v1[0].z ^ v1[1].z) ^ (v1[2].z ^ v1[3].z);
                    m[7] ^= (v1[0].w ^ v1[1].w) ^ (v1[2].w ^ v1[3].w);
                    tm_st8(ta, m);
                }
            }
        };

        // prologue: sets s0 .. s0+2 in flight, T(s0) built, query words of s0 loading
        uint4 wn[NQ];
        load_q(s0, wn);
#pragma unroll
        for (int p = 0; p < Q_NST - 1; ++p) {
            if (s0 + p < s1) stage(s0 + p, seq0 + p);
            cp_async_commit();
        }
        cp_async_wait<Q_NST - 3>();
        __syncthreads();
        build(int(seq0 % Q_NST), int(seq0 & 1));
        __syncthreads();
#pragma unroll 1
        for (uint32_t j = s0; j < s1; ++j) {
            const uint32_t sq = seq0 + (j - s0);
            uint4 wc[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) wc[q] = wn[q];
            if (j + 1 < s1) load_q(j + 1, wn);
            if (j + Q_NST - 1 < s1) stage(j + Q_NST - 1, sq + Q_NST - 1);
            cp_async_commit();
            if (j + 1 < s1) build(int((sq + 1) % Q_NST), int((sq + 1) & 1));
            lookups(wc, int(sq & 1));
            tm_wait_st();
            cp_async_wait<Q_NST - 3>();
            __syncthreads();
        }
        seq0 += s1 - s0;

        // flush: lane i holds half (i&1) of its 32-byte slice in m[0..3]. Without
        // peers (or with one segment per tile) the slice goes straight to its row;
        // with peers and several segments it goes to the local partial buffer and
        // the tile's last segment pushes the finished rows to their owners.
        const bool to_partial = peers.n && n_seg > 1;
#pragma unroll 1
        for (int s = 0; s < 4 * NQ; ++s) {
            uint32_t m[8];
            tm_ld8(tcol + 8 * s, m);
            tm_wait_ld8(m);
            const uint32_t rl = 4 * uint32_t((s >> 2) * Q_NT + tid) + uint32_t(s & 3);
            const uint32_t r = r_base + rl;
            if (r < B) {
                uint8_t* const base = to_partial ? peers.partial : peers.n ? peers.owner_out(r) : out;
                uint8_t* o = base + uint64_t(r) * S + uint64_t(c) * 32;
                uint8_t* oa = o + 16 * (i8 & 1);
                uint8_t* ob = o + 16 * ((i8 & 1) ^ 1);
                if (peers.n && !to_partial) {  // owners' rows take every rank's partials: system scope
                    red_xor64_sys(oa, uint64_t(m[1]) << 32 | m[0]);
                    red_xor64_sys(oa + 8, uint64_t(m[3]) << 32 | m[2]);
                    red_xor64_sys(ob, uint64_t(m[5]) << 32 | m[4]);
                    red_xor64_sys(ob + 8, uint64_t(m[7]) << 32 | m[6]);
                } else {
                    red_xor64(oa, uint64_t(m[1]) << 32 | m[0]);
                    red_xor64(oa + 8, uint64_t(m[3]) << 32 | m[2]);
                    red_xor64(ob, uint64_t(m[5]) << 32 | m[4]);
                    red_xor64(ob + 8, uint64_t(m[7]) << 32 | m[6]);
                }
            }
        }
        if (to_partial) {
            // arrival (threadFenceReduction pattern): every thread's REDs are ordered
            // before thread 0's count; the last arriver sees all segments' REDs
            volatile uint32_t* last = reinterpret_cast<volatile uint32_t*>(smem + C::OFF_ADDR + 4);
            __threadfence();
            __syncthreads();
            if (tid == 0) *last = atomicAdd(peers.tile_cnt + uint64_t(rt) * n_ctiles + c, 1u) == n_seg - 1;
            __syncthreads();
            if (*last) {
                __threadfence();
                unsigned long long remote = 0, own = 0;
                const uint32_t rows = (B - r_base) < uint32_t(C::RC) ? B - r_base : uint32_t(C::RC);
#pragma unroll 1
                for (uint32_t rl = tid; rl < rows; rl += Q_NT) {
                    const uint32_t r = r_base + rl;
                    uint4* p = reinterpret_cast<uint4*>(peers.partial + uint64_t(r) * S + uint64_t(c) * 32);
                    const uint4 a = __ldcg(p), b = __ldcg(p + 1);
                    __stcg(p, make_uint4(0, 0, 0, 0));
                    __stcg(p + 1, make_uint4(0, 0, 0, 0));
                    const uint32_t g = peers.owner(r);
                    uint8_t* o = peers.ptr[g] + uint64_t(r) * S + uint64_t(c) * 32;
                    red_xor64_sys(o, uint64_t(a.y) << 32 | a.x);
                    red_xor64_sys(o + 8, uint64_t(a.w) << 32 | a.z);
                    red_xor64_sys(o + 16, uint64_t(b.y) << 32 | b.x);
                    red_xor64_sys(o + 24, uint64_t(b.w) << 32 | b.z);
                    if (g == peers.self) own += 32; else remote += 32;
                }
                if (peers.stats) {
                    remote = __reduce_add_sync(0xffffffffu, uint32_t(remote));
                    own = __reduce_add_sync(0xffffffffu, uint32_t(own));
                    if (lane == 0 && remote) atomicAdd(peers.stats, remote);
                    if (lane == 0 && own) atomicAdd(peers.stats + 1, own);
                }
                if (tid == 0) peers.tile_cnt[uint64_t(rt) * n_ctiles + c] = 0;  // ready for the next launch
            }
            __syncthreads();  // the flag is rewritten by the next unit
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase), "n"(C::TCOLS));
}

namespace {

template <int NQ>
cudaError_t launch_q(const M4Args& a, int num_sms) {
    using C = QCfg<NQ>;
    cudaError_t e = cudaFuncSetAttribute(k_scan_m4rm_q<NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    const uint32_t n_ctiles = a.S / 32;
    const uint32_t n_rtiles = (a.B + C::RC - 1) / C::RC;
    const uint32_t n_groups = (a.nb + 7) / 8;
    const uint32_t n_sets = (n_groups + 3) / 4;
    // Segments per (request tile, column tile): about 32 units per CTA and, when
    // the shapes allow, a unit count that is a multiple of the grid (config 4:
    // 128 column tiles x 37 segments = 32 x 148); segments of >= 32 sets.
    const uint64_t pairs = uint64_t(n_ctiles) * n_rtiles;
    const uint64_t grid = uint64_t(num_sms);
    uint64_t x = pairs, y = grid;
    while (y) {
        const uint64_t t = x % y;
        x = y;
        y = t;
    }
    const uint64_t step = grid / x;
    const uint64_t target = (32 * grid + pairs - 1) / pairs;
    uint64_t n_seg = (target + step - 1) / step * step;
    if (step > 4 * target) n_seg = target;
    const uint64_t max_seg = n_sets / 32 > 0 ? n_sets / 32 : 1;
    if (n_seg > max_seg) n_seg = max_seg;
    if (n_seg < 1) n_seg = 1;
    k_scan_m4rm_q<NQ><<<dim3(uint32_t(grid)), Q_NT, C::SMEM, a.stream>>>(
        a.db, a.nb, a.S, a.qT, a.qstride, a.B, a.out, n_ctiles, n_sets, uint32_t(n_seg), a.peers);
    return cudaGetLastError();
}

}  // namespace

// Modelled time of a batch (arbitrary units: padded requests / measured
// efficiency) for each tile size; the efficiencies are measured fractions of the
// dense-ALU roofline at full tiles on a 1 GiB store (prof_m4rm_tiles.py):
// 2048 -> 2.89, 4096 -> 3.21, 8192 -> 3.38 (the half-TMEM 128-byte-column kernel: 3.0).
double m4rm_q_cost(uint32_t B, int* tile) {
    static const int rcs[3] = {2048, 4096, 8192};
    static const double eff[3] = {2.89, 3.21, 3.38};
    double best = 1e300;
    int best_rc = 2048;
    for (int k = 0; k < 3; ++k) {
        const double cost = double((uint64_t(B) + rcs[k] - 1) / rcs[k] * rcs[k]) / eff[k];
        if (cost < best * 0.999) {
            best = cost;
            best_rc = rcs[k];
        }
    }
    if (tile) *tile = best_rc;
    return best;
}

int m4rm_q_tile(uint32_t B) {
    int t = 2048;
    m4rm_q_cost(B, &t);
    return t;
}

cudaError_t launch_scan_m4rm_q(const M4Args& a, int num_sms) {
    if (a.S % 32 != 0) return cudaErrorInvalidValue;
    switch (m4rm_q_tile(a.B)) {
        case 8192: return launch_q<4>(a, num_sms);
        case 4096: return launch_q<2>(a, num_sms);
        default: return launch_q<1>(a, num_sms);
    }
}

}  // namespace xpir
