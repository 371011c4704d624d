// K1q (kernel 8, B >= 4096 and S % 32 == 0): M4RM with 9-bucket tables over
// 32-byte columns, four tables interleaved per bank line, accumulators entirely
// in Tensor Memory — the headline scan.
//
// Same math as every M4RM kernel: T[x] = XOR of the buckets selected by the bits
// of x, the answer slice of request r is the XOR over tables of T[index_r]
// (bit-exact pir::answer_batch, pir.cpp:41-52). Round 1's K1q used 8-bucket
// (byte) tables; round 2 replaced it with this kernel (profiles/r02_ncu_m4rm_q9_summary.txt:
// 123.3 against 136.8 ms per config-4 launch, bit-exact). What changed:
//
//  * A table covers 9 buckets (512 rows of 32 bytes), so one lookup serves 9
//    buckets instead of 8: the lookup wavefronts per bucket drop by 1/9.
//  * A *pair* is 72 buckets = 9 query bytes. Query bytes 0..7 of a pair are the
//    low 8 index bits of the pair's eight tables (two sets of four); byte 8
//    holds their ninth bits (nibble h of the byte for set h). So set h of pair p
//    = tables t = 0..3 over buckets 72p + 32h + 8t + i (i < 8, bit i of query
//    byte 9p + 4h + t) and 72p + 64 + 4h + t (bit 4h + t of query byte 9p + 8).
//    The query layout is a pure byte permutation of the PIR bit vector
//    (k_expand_T / k_transpose_q layout 2): low bytes in the set-interleaved
//    32-bit words K1q reads, the ninth-bit bytes in a plane after them
//    ([pair][request] bytes, four requests per 32-bit load).
//  * Four 512-row tables of a set interleave per 128-byte bank line exactly as in
//    K1q (row x of table t at x*128 + 32t): one set = 64 KiB, double-buffered
//    128 KiB. The 9-bit index is one PRMT of the set word and the request's ninth
//    bits spread to one byte per table (IMAD by 0x204081 + LOP3, once per
//    request and set).
//  * Shared-memory wavefronts per set (Rc = 8192): 8192 lookups + 512 table
//    stores + 144 bucket-word reads + 256 + 32 index loads + ~10 staging fills
//    = 9146 per 36 buckets, against K1q's 8776 per 32 buckets: 7% fewer per
//    bucket. The index costs what the byte tables' did (PRMT + IMAD per lookup)
//    plus three instructions per request and set.
//
// Unchanged from the byte-table version:
//  * One lane owns one request and its full 32-byte slice (two 16-byte halves).
//    In step kk of a set, lane i of a quarter-warp reads table
//    t = ((i>>1) + kk) & 3, half (i&1) first: the eight lanes of a quarter-warp
//    always hit eight distinct 16-byte bank groups, so every LDS.128 is a single
//    conflict-free wavefront per quarter-warp, for any query bytes.
//  * Accumulators: 32 bytes x 16 requests per thread = all 256 KiB of TMEM
//    (tcgen05.ld/st .32x32b.x8), read-modify-written once per set. Rc = 8192
//    requests per tile (templated 2048 / 4096 / 8192).
//  * Index words are read straight from L2 into registers one set ahead (LDG with
//    an L2 evict_last policy), bucket slices staged by cp.async (zero-fill past the
//    shard, evict_first) three sets ahead; the build of set j+1 overlaps the
//    lookups of set j (double-buffered tables).
//  * Segment partials XOR into the answer rows (red.xor with an evict_last policy,
//    so DRAM sees each answer row once), or, for the fused cross-GPU reduce, into a
//    local partial buffer whose last-arriving segment pushes each finished row to
//    its owner rank over NVLink (red.relaxed.sys).
//
// Pipeline without CTA barriers: every warp builds 32 of a set's 512 table rows
// and then looks up its own requests. Per table buffer two mbarriers — full[b]
// (all 16 warps have written their rows of the set in b) and empty[b] (all 16
// have finished its lookups) — and per staging slot one mbarrier that the
// cp.async copies of the bucket slices arrive on as they land. A warp waits only
// for what it reads next, so warps drift up to a set apart instead of meeting at
// a barrier per set (config 4: 128.4 ms with a barrier per set -> 123.3 ms; the
// 2048/4096-request tiles 5% / 3% faster).
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

constexpr int R_NT = 512;
constexpr int R_TAB = 512 * 128;  // one set of four interleaved 512-row tables
constexpr int R_NST = 4;          // staging ring depth (sets)
constexpr int R_STG = 36 * 32;    // 36 buckets x 32 B per staged set

template <int NQ>
struct RCfg {
    static constexpr int RC = R_NT * 4 * NQ;  // requests per tile
    // two table buffers, staging ring, TMEM slot
    static constexpr int OFF_STG = 2 * R_TAB;
    static constexpr int OFF_ADDR = OFF_STG + R_NST * R_STG;
    static constexpr int OFF_MBAR = OFF_ADDR + 16;  // full[2], empty[2], staged[R_NST]
    static constexpr int SMEM = OFF_MBAR + 32 + 8 * R_NST;
    static constexpr int TCOLS = 128 * NQ;
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
__device__ __forceinline__ void tm_wait_ld8(uint32_t (&v)[8]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;\n"
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]),
                   "+r"(v[7])
                 :
                 : "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ uint4 ldg_q(const uint8_t* p, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;\n"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint32_t ldg_h(const uint8_t* p, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;\n" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
// store slices stream through L2 once: evict_first, so they do not push out the
// shared index words or the answer rows
__device__ __forceinline__ void cp_async16_ef(uint32_t dst, const void* src, uint32_t src_bytes, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;\n" ::"r"(dst), "l"(src),
                 "r"(src_bytes), "l"(pol));
}
// segment flushes XOR into answer rows that every segment of the tile revisits:
// evict_last keeps the rows in L2 between segments (DRAM sees them once)
__device__ __forceinline__ void red_xor64_el(void* p, uint64_t v, uint64_t pol) {
    asm volatile("red.relaxed.gpu.global.xor.L2::cache_hint.b64 [%0], %1, %2;\n" ::"l"(p), "l"(v), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared.b64 st, [%0];\n}\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}
// the mbarrier counts this thread's prior cp.async copies as they land (.noinc:
// the barrier's expected count, set at init, already includes them)
__device__ __forceinline__ void cp_async_mbar_arrive(uint32_t a) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
    return pol;
}

}  // namespace

// qT: low index bytes, set-interleaved ([set][request] 32-bit words, 2 sets per
// pair); qH: ninth-bit bytes ([pair][request]). Both qstride requests wide.
template <int NQ>
__global__ void __launch_bounds__(R_NT, 1)
k_scan_m4rm_q9(const uint8_t* __restrict__ db, uint32_t nb, uint32_t S, const uint8_t* __restrict__ qT,
               const uint8_t* __restrict__ qH, uint64_t qstride, uint32_t B, uint8_t* __restrict__ out,
               uint32_t n_ctiles, uint32_t n_pairs, uint32_t n_seg, PeerOut peers) {
    using C = RCfg<NQ>;
    extern __shared__ __align__(1024) uint8_t smem[];
    const uint32_t sbase = smem_u32(smem);
    uint8_t* const sgen = smem;
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
    const uint32_t tbase = *reinterpret_cast<const uint32_t*>(sgen + C::OFF_ADDR);
    // mbarriers: full[b] / empty[b] per table buffer (16 warp arrivals each),
    // staged[k] per staging slot (72 copying threads' cp.async completions)
    const uint32_t mb_full = sbase + C::OFF_MBAR, mb_empty = sbase + C::OFF_MBAR + 16,
                   mb_stg = sbase + C::OFF_MBAR + 32;
    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(mb_full + 8 * b, 16);
            mbar_init(mb_empty + 8 * b, 16);
        }
        for (int b = 0; b < R_NST; ++b) mbar_init(mb_stg + 8 * b, 72);
    }
    __syncthreads();
    const uint32_t tcol = tbase + (uint32_t((warp & 3) * 32) << 16) + uint32_t(warp >> 2) * (32 * NQ);

    // lookup constants: step kk reads table t = (lp + kk) & 3, own half first
    uint32_t toff[4], bsel[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
        const uint32_t t = uint32_t(lp + kk) & 3u;
        toff[kk] = 32 * t + 16 * uint32_t(i8 & 1);
        // 9-bit index in one PRMT: byte 0 = low byte t of the set word, byte 1 =
        // byte t of the spread ninth bits (0/1), bytes 2-3 = sign of that byte (0)
        bsel[kk] = t | ((4u + t) << 4) | ((12u + t) << 8) | ((12u + t) << 12);
    }
    const uint32_t dhalf = (i8 & 1) ? 0xfffffff0u : 16u;
    // build constants: lane -> (table bt, 32-bit word bw); warp -> index bits 4..7
    const int bt = lane >> 3, bw = lane & 7;
    const uint32_t hm0 = 0u - (warp & 1u), hm1 = 0u - ((warp >> 1) & 1u), hm2 = 0u - ((warp >> 2) & 1u),
                   hm3 = 0u - ((warp >> 3) & 1u);

    const uint32_t n_rtiles = (B + C::RC - 1) / C::RC;
    const uint64_t units = uint64_t(n_ctiles) * n_rtiles * n_seg;
    uint32_t seq0 = 0;  // staging sequence number (always even at a unit start)

    for (uint64_t v = blockIdx.x; v < units; v += gridDim.x) {
        const uint32_t c = uint32_t(v % n_ctiles);
        const uint32_t rt = uint32_t((v / n_ctiles) % n_rtiles);
        const uint32_t sg = uint32_t(v / (uint64_t(n_ctiles) * n_rtiles));
        const uint32_t p0 = uint32_t(uint64_t(n_pairs) * sg / n_seg);
        const uint32_t p1 = uint32_t(uint64_t(n_pairs) * (sg + 1) / n_seg);
        if (p0 >= p1) continue;
        const uint32_t s0 = 2 * p0, s1 = 2 * p1;
        const uint32_t r_base = rt * C::RC;

        {
            uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
            for (int s = 0; s < 4 * NQ; ++s) tm_st8(tcol + 8 * s, z);
            tm_wait_st();
        }

        // set j: pair j/2, half j&1; staged [i][t][32 B], i = 8 is the ninth bucket
        const uint64_t qpol = l2_evict_last_policy(), spol = l2_evict_first_policy();
        auto stage = [&](uint32_t j, uint32_t sq) {
            const int buf = int(sq % R_NST);
            const uint32_t dst = sbase + C::OFF_STG + buf * R_STG;
            if (tid < 72) {
                const uint32_t i = tid >> 3, t = (tid >> 1) & 3, part = tid & 1;
                const uint32_t p = j >> 1, h = j & 1;
                const uint32_t bucket = i < 8 ? 72 * p + 32 * h + 8 * t + i : 72 * p + 64 + 4 * h + t;
                const bool ok = bucket < nb;
                const uint8_t* src = db + (ok ? uint64_t(bucket) * S : 0) + uint64_t(c) * 32 + part * 16;
                cp_async16_ef(dst + tid * 16, src, ok ? 16u : 0u, spol);
                cp_async_mbar_arrive(mb_stg + 8 * buf);
            }
        };
        auto load_q = [&](uint32_t j, uint4 (&w)[NQ]) {
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const uint32_t r4 = r_base + 4 * uint32_t(q * R_NT + tid);
                w[q] = r4 < qstride ? ldg_q(qT + uint64_t(j) * 4 * qstride + uint64_t(r4) * 4, qpol)
                                    : make_uint4(0, 0, 0, 0);
            }
        };
        auto load_h = [&](uint32_t p, uint32_t (&hw)[NQ]) {
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const uint32_t r4 = r_base + 4 * uint32_t(q * R_NT + tid);
                hw[q] = r4 < qstride ? ldg_h(qH + uint64_t(p) * qstride + r4, qpol) : 0u;
            }
        };
        // Warps 0-7 build: warp w writes the rows whose index bits 4..6 equal w, for
        // the four values of bits 7..8 (16 Gray-code rows over buckets 0..3 each).
        // (All 16 warps building two blocks each measured no faster.)
        // warp w writes the rows whose index bits 4..7 equal w, for both values of
        // bit 8 (two 16-row Gray-code blocks over buckets 0..3)
        auto build = [&](int buf, int tb) {
            const uint32_t src = sbase + C::OFF_STG + buf * R_STG + bt * 32 + bw * 4;
            uint32_t b[9];
#pragma unroll
            for (int i = 0; i < 9; ++i) b[i] = lds32(src + i * 128);
            const uint32_t h = (b[4] & hm0) ^ (b[5] & hm1) ^ (b[6] & hm2) ^ (b[7] & hm3);
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const uint32_t row0 = sbase + tb * R_TAB + uint32_t((warp + 16 * u) << 4) * 128 + bt * 32 + bw * 4;
                uint32_t x = h ^ (u ? b[8] : 0u);
                sts32(row0, x);
#pragma unroll
                for (int m = 1; m < 16; ++m) {
                    x ^= b[(m & 1) ? 0 : (m & 2) ? 1 : (m & 4) ? 2 : 3];  // ctz(m)
                    sts32(row0 + uint32_t(m ^ (m >> 1)) * 128, x);
                }
            }
        };
        auto lookups = [&](const uint4 (&wq)[NQ], const uint32_t (&hq)[NQ], const uint32_t hshift, int tb) {
            uint32_t tk[4];
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) tk[kk] = sbase + tb * R_TAB + toff[kk];
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const uint32_t wk[4] = {wq[q].x, wq[q].y, wq[q].z, wq[q].w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t ta = tcol + 8 * (4 * q + k);
                    uint32_t m[8];
                    tm_ld8(ta, m);
                    // ninth bits of the request's four tables -> bytes 0..3 (bit t -> bit 8t)
                    const uint32_t hx = (((hq[q] >> (8 * k + hshift)) & 15u) * 0x204081u) & 0x01010101u;
                    uint4 v0[4], v1[4];
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        uint32_t i9;  // PTX prmt (not __byte_perm): selector bit 3 = sign-replicate
                        asm("prmt.b32 %0, %1, %2, %3;" : "=r"(i9) : "r"(wk[k]), "r"(hx), "r"(bsel[kk]));
                        const uint32_t a0 = i9 * 128 + tk[kk];
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

        // prologue: sets s0 .. s0+2 in flight, words of s0 and pair p0 loading, T(s0) built
        uint4 wn[NQ];
        uint32_t hn[NQ], hc[NQ];
        load_q(s0, wn);
        load_h(p0, hn);
#pragma unroll
        for (int p = 0; p < R_NST - 1; ++p)
            if (s0 + p < s1) stage(s0 + p, seq0 + p);
        mbar_wait(mb_stg + 8 * (seq0 % R_NST), (seq0 / R_NST) & 1);
        if (seq0) mbar_wait(mb_empty, ((seq0 >> 1) - 1) & 1);
        build(int(seq0 % R_NST), 0);
        __syncwarp();
        if (lane == 0) mbar_arrive(mb_full);
#pragma unroll 1
        for (uint32_t jp = s0; jp < s1; jp += 2) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {  // table buffer = h (seq0 is even)
                const uint32_t j = jp + h;
                const uint32_t sq = seq0 + (j - s0);
                uint4 wc[NQ];
#pragma unroll
                for (int q = 0; q < NQ; ++q) wc[q] = wn[q];
                if (h == 0) {
#pragma unroll
                    for (int q = 0; q < NQ; ++q) hc[q] = hn[q];
                }
                if (j + 1 < s1) {
                    load_q(j + 1, wn);
                    if (h == 1) load_h((j + 1) >> 1, hn);
                }
                if (j + R_NST - 1 < s1) stage(j + R_NST - 1, sq + R_NST - 1);
                if (j + 1 < s1) {  // this warp's rows of set j+1, once its slices landed and buffer h^1 is free
                    const uint32_t sb = sq + 1;
                    mbar_wait(mb_stg + 8 * (sb % R_NST), (sb / R_NST) & 1);
                    mbar_wait(mb_empty + 8 * (h ^ 1), ((sb >> 1) - 1) & 1);
                    build(int(sb % R_NST), h ^ 1);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(mb_full + 8 * (h ^ 1));
                }
                mbar_wait(mb_full + 8 * h, (sq >> 1) & 1);  // set j built by every warp
                lookups(wc, hc, 4u * uint32_t(h), h);
                tm_wait_st();
                __syncwarp();
                if (lane == 0) mbar_arrive(mb_empty + 8 * h);
            }
        }
        seq0 += s1 - s0;
        __syncthreads();  // the next unit restages and rebuilds

        // flush (K1q's): straight to the rows, or through the local partial buffer
        // and the tile's last segment when the fused cross-GPU reduce is on
        const bool to_partial = peers.n && n_seg > 1;
#pragma unroll 1
        for (int s = 0; s < 4 * NQ; ++s) {
            uint32_t m[8];
            tm_ld8(tcol + 8 * s, m);
            tm_wait_ld8(m);
            const uint32_t rl = 4 * uint32_t((s >> 2) * R_NT + tid) + uint32_t(s & 3);
            const uint32_t r = r_base + rl;
            if (r < B) {
                uint8_t* const base = to_partial ? peers.partial : peers.n ? peers.owner_out(r) : out;
                uint8_t* o = base + uint64_t(r) * S + uint64_t(c) * 32;
                uint8_t* oa = o + 16 * (i8 & 1);
                uint8_t* ob = o + 16 * ((i8 & 1) ^ 1);
                if (peers.n && !to_partial) {
                    red_xor64_sys(oa, uint64_t(m[1]) << 32 | m[0]);
                    red_xor64_sys(oa + 8, uint64_t(m[3]) << 32 | m[2]);
                    red_xor64_sys(ob, uint64_t(m[5]) << 32 | m[4]);
                    red_xor64_sys(ob + 8, uint64_t(m[7]) << 32 | m[6]);
                } else {
                    red_xor64_el(oa, uint64_t(m[1]) << 32 | m[0], qpol);
                    red_xor64_el(oa + 8, uint64_t(m[3]) << 32 | m[2], qpol);
                    red_xor64_el(ob, uint64_t(m[5]) << 32 | m[4], qpol);
                    red_xor64_el(ob + 8, uint64_t(m[7]) << 32 | m[6], qpol);
                }
            }
        }
        if (to_partial) {
            volatile uint32_t* last = reinterpret_cast<volatile uint32_t*>(sgen + C::OFF_ADDR + 4);
            __threadfence();
            __syncthreads();
            if (tid == 0) *last = atomicAdd(peers.tile_cnt + uint64_t(rt) * n_ctiles + c, 1u) == n_seg - 1;
            __syncthreads();
            if (*last) {
                __threadfence();
                unsigned long long remote = 0, own = 0;
                const uint32_t rows = (B - r_base) < uint32_t(C::RC) ? B - r_base : uint32_t(C::RC);
#pragma unroll 1
                for (uint32_t rl = tid; rl < rows; rl += R_NT) {
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
                if (tid == 0) peers.tile_cnt[uint64_t(rt) * n_ctiles + c] = 0;
            }
            __syncthreads();
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
cudaError_t launch_q9(const M4Args& a, int num_sms) {
    using C = RCfg<NQ>;
    cudaError_t e = cudaFuncSetAttribute(k_scan_m4rm_q9<NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    const uint32_t n_ctiles = a.S / 32;
    const uint32_t n_rtiles = (a.B + C::RC - 1) / C::RC;
    const uint32_t n_pairs = (a.nb + 71) / 72;
    // segments per (request tile, column tile): K1q's rule (about 32 units per CTA,
    // a unit count that is a multiple of the grid when the shapes allow), in pairs
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
    const uint64_t max_seg = n_pairs / 16 > 0 ? n_pairs / 16 : 1;
    if (n_seg > max_seg) n_seg = max_seg;
    // and segments short enough that the index bytes a wave of CTAs shares
    // (pairs x 9 B x Rc) stay near 7.5 MiB: measured at config 4, 148 segments
    // (98 pairs each) 130.5 ms against 133.3 ms for 37; 1 GiB stores are there already
    const uint64_t want = (uint64_t(n_pairs) * 9 * C::RC + (15u << 19) - 1) / (15u << 19);
    if (n_seg < want) n_seg = step <= want ? (want + step - 1) / step * step : want;
    if (n_seg < 1) n_seg = 1;
    const uint8_t* qH = a.qT + m4rm_q9_hi_offset(a.nb, a.qstride);
    k_scan_m4rm_q9<NQ><<<dim3(uint32_t(grid)), R_NT, C::SMEM, a.stream>>>(
        a.db, a.nb, a.S, a.qT, qH, a.qstride, a.B, a.out, n_ctiles, n_pairs, uint32_t(n_seg), a.peers);
    return cudaGetLastError();
}

}  // namespace

// Modelled time of a batch (arbitrary units: padded requests / measured
// efficiency) for each tile size; the efficiencies are measured fractions of the
// dense-ALU roofline at full tiles on a 1 GiB store, S = 4096 (scripts/time_scan.py):
// 2048 -> 2.96, 4096 -> 3.46, 8192 -> 3.80 (the half-TMEM 128-byte-column kernel:
// 3.0, still 1-2% faster at B = 2048 and 6144).
double m4rm_q_cost(uint32_t B, int* tile) {
    static const int rcs[3] = {2048, 4096, 8192};
    static const double eff[3] = {2.96, 3.46, 3.80};
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

uint64_t m4rm_q9_hi_offset(uint32_t nb, uint64_t qstride) { return uint64_t((nb + 71) / 72) * 8 * qstride; }

cudaError_t launch_scan_m4rm_q(const M4Args& a, int num_sms) {
    if (a.S % 32 != 0) return cudaErrorInvalidValue;
    switch (m4rm_q_tile(a.B)) {
        case 8192: return launch_q9<4>(a, num_sms);
        case 4096: return launch_q9<2>(a, num_sms);
        default: return launch_q9<1>(a, num_sms);
    }
}

}  // namespace xpir
