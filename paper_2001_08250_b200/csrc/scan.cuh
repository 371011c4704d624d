// Launch interfaces of the scan kernels (scan.cu) and write-path kernels (write.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace xpir {

constexpr uint32_t XPIR_MAX_DISPLACEMENTS_DEV = 500;  // cuckoo.hpp:15

// Count of kernels launched through the library (reported as gpu_launches).
void count_launches(uint64_t n);

struct ScanArgs {
    const uint8_t* db;   // shard, bucket-major, nb * S bytes
    uint32_t nb;         // buckets in the shard
    uint32_t S;          // bucket bytes
    const uint8_t* q;    // query rows, already offset to the shard's first byte
    uint64_t q_stride;   // bytes between rows
    uint32_t B;          // requests
    uint8_t* out;        // B * S, pre-initialised (zero or mask pad); scan XORs into it
    cudaStream_t stream;
};

// Fused cross-GPU reduction target: answer row r belongs to the rank g with
// bound[g] <= r < bound[g+1]; every rank's buffer holds all B rows at the same
// offsets (only the owner's rows are meaningful). n == 0: no peers.
// Fused cross-GPU reduce of the quad-table scan (m4rm_q9.cu): rank g owns answer
// rows [bound[g], bound[g+1]) in its buffer ptr[g] (CUDA-IPC peer pointers).
// Segment partials of one (request tile, column tile) accumulate in this GPU's
// `partial` buffer; the last segment to arrive (tile_cnt) pushes the tile's rows
// to their owners once — B*S bytes per rank per batch, (G-1)/G of them remote.
// partial and tile_cnt are zero between launches (the pusher clears its tile).
struct PeerOut {
    uint8_t* ptr[8];
    uint32_t bound[9];
    uint32_t n;
    uint32_t self;                      // this rank
    uint8_t* partial;                   // B x S local accumulation buffer
    uint32_t* tile_cnt;                 // arrivals per (request tile, column tile)
    unsigned long long* stats;          // [0] remote bytes pushed, [1] own-row bytes (nullable)
    __device__ __forceinline__ uint32_t owner(uint32_t r) const {
        uint32_t g = 0;
#pragma unroll
        for (int k = 1; k < 8; ++k)
            if (k < int(n) && r >= bound[k]) g = k;
        return g;
    }
    __device__ __forceinline__ uint8_t* owner_out(uint32_t r) const { return ptr[owner(r)]; }
};

// M4RM scan (m4rm.cu): queries in the group-major layout qT[g*qstride + r].
struct M4Args {
    const uint8_t* db;
    uint32_t nb, S;
    const uint8_t* qT;
    uint64_t qstride;    // multiple of 16, >= B
    uint32_t B;
    uint8_t* out;
    cudaStream_t stream;
    PeerOut peers{};     // set only by the sharded fused path (TMEM kernel)
};
cudaError_t launch_scan_m4rm(const M4Args& a, int ctas_per_sm, int num_sms, int variant);
cudaError_t launch_scan_m4rm_tmem(const M4Args& a, int num_sms);
// quad-interleaved 9-bucket tables over 32-byte columns, full-TMEM accumulators
// (m4rm_q9.cu, kernel 8); S % 32 == 0; queries in layout 2
cudaError_t launch_scan_m4rm_q(const M4Args& a, int num_sms);
int m4rm_q_tile(uint32_t B);
uint64_t m4rm_q9_hi_offset(uint32_t nb, uint64_t qstride);
double m4rm_q_cost(uint32_t B, int* tile);  // vs the half-TMEM kernel: ceil(B/2048)*2048/3.0
cudaError_t launch_scan_m4rm4(const M4Args& a, int num_sms);  // nibble tables (m4rm4.cu)
cudaError_t launch_scan_m4rm6(const M4Args& a, int num_sms);  // 6-bucket tables (m4rm6.cu)
uint64_t m4rm_qstride(uint32_t B);
uint64_t m4rm_qrows(uint64_t n_groups);  // rows to allocate (staging reads 16-row chunks)
// layout: see m4rm_layout below (k_expand_T runs k_expand_q9 for layout 2)
cudaError_t launch_expand_T(const uint8_t* seeds, uint32_t B, uint64_t byte_lo, uint64_t nbytes,
                            uint8_t* qT, uint64_t qstride, cudaStream_t s, int layout = 0);
cudaError_t launch_transpose_q(const uint8_t* q, uint64_t q_stride, uint64_t byte_lo, uint64_t nbytes,
                               uint32_t B, uint8_t* qT, uint64_t qstride, cudaStream_t s, int layout = 0);
// query layout each M4RM kernel reads: 0 group-major bytes (kernels 2/5/7/9),
// 2 pairs of 9-bucket sets (kernel 8)
inline int m4rm_layout(int kernel) { return kernel == 8 ? 2 : 0; }
cudaError_t launch_scan_direct(const ScanArgs& a, int num_sms, uint32_t* nsplit_out);
cudaError_t launch_scan_bytes(const ScanArgs& a);
cudaError_t launch_init_out(uint8_t* out, uint32_t B, uint32_t S, const uint8_t* mask_seeds,
                            bool xor_into, cudaStream_t s);
cudaError_t launch_expand(const uint8_t* seeds, uint32_t B, uint64_t byte_lo, uint64_t nbytes,
                          uint8_t* qout, uint64_t stride, cudaStream_t s, const uint32_t* rows = nullptr);
cudaError_t launch_scatter_rows(const uint8_t* src, uint64_t ss, uint32_t n, const uint32_t* idx, uint8_t* dst,
                                uint64_t ds, uint64_t nbytes, cudaStream_t s);
cudaError_t launch_xor_reduce(uint8_t* dst, const uint8_t* const* d_srcs, uint32_t nsrc,
                              uint64_t bytes, int num_sms, cudaStream_t s);
cudaError_t run_peak_kernels(int num_sms, double* lop3_per_s, double* smem_bps, cudaStream_t s);
cudaError_t run_tmem_probe(int variant, int num_sms, double* bytes_per_clk_sm);

// write path / generators (write.cu)
cudaError_t launch_keystream(const uint8_t* key_host32, uint64_t nonce, uint64_t byte_offset,
                             uint8_t* out, uint64_t len, cudaStream_t s);
cudaError_t launch_keystream_rows(const uint8_t* key_host32, uint64_t nonce0, uint32_t rows,
                                  uint64_t len, uint8_t* out, uint64_t row_stride, cudaStream_t s);
cudaError_t launch_prf2(const uint64_t k1[2], const uint64_t k2[2], const uint64_t* in, uint64_t n,
                        uint64_t modulus, uint32_t* o1, uint32_t* o2, cudaStream_t s);
cudaError_t launch_prf(uint64_t k0, uint64_t k1, const uint64_t* in, uint64_t n, uint64_t modulus,
                       uint64_t* out, uint32_t* out32, cudaStream_t s);
cudaError_t launch_interest(const uint8_t* id16_host, const uint64_t* seqs, uint64_t n, uint32_t h,
                            uint32_t m_bits, uint32_t* pos_out, unsigned long long* words,
                            cudaStream_t s);
cudaError_t launch_bloom_item(const uint8_t* item_dev, uint32_t len, uint32_t h, uint32_t m_bits,
                              uint32_t* out, cudaStream_t s);
// scratch: 8 bytes of device memory; on return it holds the index of the first
// out-of-range position (or ~0); positions before it are absorbed (notify.cpp:60-65).
cudaError_t launch_absorb(const uint32_t* pos, uint64_t n, uint32_t m_bits,
                          unsigned long long* words, unsigned long long* scratch, cudaStream_t s);
cudaError_t launch_absorb_unchecked(const uint32_t* pos, uint64_t n, unsigned long long* words, cudaStream_t s);
// first index whose beta1 or beta2 >= buckets into *first_bad (~0 when none)
cudaError_t launch_beta_check(const uint32_t* b1, const uint32_t* b2, uint64_t n, uint32_t buckets,
                              unsigned long long* first_bad, cudaStream_t s);
cudaError_t launch_draws(const uint8_t* key_host32, uint64_t nonce0, uint32_t count, uint64_t* out,
                         cudaStream_t s);

// Interest-delta codecs (codec.cu): notify::encode_delta / decode_delta.
size_t encode_delta_scratch_bytes(uint64_t nwords);
size_t decode_delta_scratch_bytes(uint64_t len);
cudaError_t launch_encode_delta(const uint64_t* words, uint64_t nwords, uint32_t m_bits, uint8_t* out, uint64_t cap,
                                unsigned long long* len_out, void* scratch, size_t scratch_bytes, cudaStream_t s);
// hdr: 5 x u64 of device memory; hdr[0] = 0 ok / 1 malformed / 2 words_cap too small, hdr[1] = m
cudaError_t launch_encode_positions(const uint32_t* pos, uint32_t h, uint64_t n, uint32_t cap, uint8_t* out,
                                    uint8_t* ok, cudaStream_t s);
cudaError_t launch_decode_positions(const uint8_t* fields, uint32_t cap, uint64_t n, uint32_t* pos, uint32_t* count,
                                    cudaStream_t s);
cudaError_t launch_decode_delta(const uint8_t* buf, uint64_t len, uint64_t* words, uint64_t words_cap,
                                unsigned long long* hdr, void* scratch, size_t scratch_bytes, cudaStream_t s);

// Device-resident cuckoo metadata (one per table).
struct CuckooDev {
    uint32_t buckets, depth;
    uint64_t capacity, item;
    uint8_t* used;        // [slots]
    uint32_t* beta1;      // [slots]
    uint32_t* beta2;      // [slots]
    uint64_t* stamp;      // [slots]
    int64_t* origin;      // [slots] payload source of a slot touched this batch
    uint32_t* touched_mark;  // [slots] batch id that last touched the slot
    uint32_t* touched;    // [slots] list of touched slots this batch
    int64_t* fifo;        // ring [fifo_cap] stamp -> flat slot (or -1)
    uint64_t fifo_cap;    // power of two
    uint64_t* draws;      // [draw_cap] precomputed DetRng::next_u64 values
    uint32_t draw_cap;
    uint8_t* gather;      // [slots*item] staging for moved pre-existing payloads
    uint32_t* mod_batch;  // [slots] last round (batch id) that rewrote the slot's payload
    uint64_t* chain_pre;  // [3 * 512] pre-chain contents of an eviction chain (walk_x)
};
// buckets [lo, hi) of the table (the payload shard / store shard range)
cudaError_t launch_seal_incremental(const CuckooDev& d, uint32_t lo, uint32_t hi, uint32_t since,
                                    const uint8_t* table, uint8_t* img, int num_sms, cudaStream_t s);

// Scalars the walk reads and advances (device memory, one struct).
struct CuckooState {
    uint64_t writes, live, next_stamp, fifo_head;
    uint64_t rng_block;       // DetRng fill counter (= next draw's nonce)
    uint64_t draw_base;       // nonce of draws[0]
    uint32_t draw_count;      // valid draws in the buffer
    uint32_t n_touched;
    uint32_t batch_id;
    uint32_t status;          // 0 ok, 1 need more draws (resume_at valid), 2 fifo overflow
    uint64_t resume_at;       // first insert not yet processed
    uint32_t walked;          // a walk kernel processed inserts this batch (items may have moved)
    uint32_t pad_;
    uint64_t limit;           // inserts at or past it are never walked (first out-of-range beta)
};
// Device-side start of a walk: i0 == WALK_FROM_STATE starts at gst->resume_at
// (left there by the parallel prefix); a walk with nothing to do returns at once.
constexpr uint64_t WALK_FROM_STATE = ~0ull;
__device__ __forceinline__ bool walk_prologue(CuckooState* gst, uint64_t& i0, uint64_t& n) {
    if (i0 == WALK_FROM_STATE) i0 = *reinterpret_cast<volatile uint64_t*>(&gst->resume_at);
    const uint64_t lim = *reinterpret_cast<volatile uint64_t*>(&gst->limit);
    if (lim < n) n = lim;
    if (i0 >= n) {
        __syncthreads();
        if (threadIdx.x == 0) {
            gst->status = 0;
            gst->resume_at = n;
        }
        return false;
    }
    __syncthreads();  // every thread has read resume_at before it can change
    if (threadIdx.x == 0) gst->walked = 1;
    __syncthreads();
    return true;
}

// refill a FIFO ring of `cap` entries (a power of two) from the live slots' stamps
cudaError_t launch_fifo_rebuild(const CuckooDev& d, int64_t* ring, uint64_t cap, cudaStream_t s);
cudaError_t launch_cuckoo_walk(const CuckooDev& d, CuckooState* st, const uint32_t* beta1,
                               const uint32_t* beta2, uint64_t i0, uint64_t n, uint32_t* reports,
                               cudaStream_t s);
// warp-cooperative walks: on-chip eviction control (walk_x.cu), or global
// victim metadata (walk.cu); launch_cuckoo_walk picks the first supported
bool walk_x_supported(const CuckooDev& d);
cudaError_t launch_cuckoo_walk_x(const CuckooDev& d, CuckooState* st, const uint32_t* beta1, const uint32_t* beta2,
                                 uint64_t i0, uint64_t n, uint32_t* reports, cudaStream_t s);
bool walk_w_supported(const CuckooDev& d);
// force_global: the global-map variant even when the shared-memory maps fit (small
// batches: staging the maps costs O(slots) per launch, the global variant nothing)
cudaError_t launch_cuckoo_walk_w(const CuckooDev& d, CuckooState* st, const uint32_t* beta1, const uint32_t* beta2,
                                 uint64_t i0, uint64_t n, uint32_t* reports, cudaStream_t s,
                                 bool force_global = false);
// Bucket-range payload shards of one logical table (metadata replicated on every
// shard, each shard holds the payloads of buckets [lo[g], lo[g+1])). data[g] may
// be a CUDA-IPC-mapped peer pointer (NVLink).
struct ShardMap {
    uint32_t n;
    uint32_t lo[9];
    const uint8_t* data[8];
};
// Phase 1: stage the pre-round payloads that move INTO this shard's range (from
// any shard); phase 2 (after every shard's phase 1): write this shard's touched
// slots. The payload array `table` holds buckets [lo, hi) of this shard.
// With dev_state != null the touched count is read on device from it (the host
// copy `st` is stale; max_touched bounds the grid) — no host round trip between
// the walk and the payload moves.
cudaError_t launch_cuckoo_gather_sharded(const CuckooDev& d, const CuckooState* st, uint32_t lo, uint32_t hi,
                                         const uint8_t* table, const ShardMap& map, cudaStream_t s,
                                         CuckooState* dev_state = nullptr, uint32_t max_touched = 0,
                                         uint32_t cap = 0);
cudaError_t launch_cuckoo_scatter_sharded(const CuckooDev& d, const CuckooState* st, uint32_t lo, uint32_t hi,
                                          uint8_t* table, const uint8_t* payload, cudaStream_t s,
                                          const CuckooState* dev_state = nullptr, uint32_t max_touched = 0);

// Grow-only scratch of the parallel eviction-free prefix (cuckoo_par.cu).
struct CuckooParScratch {
    void *keys_a = nullptr, *keys_b = nullptr, *outcome = nullptr, *succ = nullptr;
    void *slot_of = nullptr, *flags = nullptr, *cub_tmp = nullptr, *rank = nullptr;
    size_t keys_a_cap = 0, keys_b_cap = 0, outcome_cap = 0, succ_cap = 0, slot_cap = 0, flags_cap = 0,
           cub_cap = 0, rank_cap = 0;
    void release() {
        for (void* p : {keys_a, keys_b, outcome, succ, slot_of, flags, cub_tmp, rank})
            if (p) cudaFree(p);
        *this = CuckooParScratch{};
    }
};
cudaError_t cuckoo_reserve(CuckooParScratch& sc, uint64_t n, uint32_t buckets, cudaStream_t s);
// Launches the parallel eviction-free prefix of a batch of n inserts on stream s,
// entirely from and into the device state `st` (no host round trip): it starts
// the batch (batch_id + 1, n_touched = 0), places the prefix, and leaves
// resume_at = prefix length, limit = first insert with a bucket out of range
// (n when none) for the walk launched after it with i0 = WALK_FROM_STATE.
cudaError_t cuckoo_parallel_prefix(const CuckooDev& d, CuckooState* st, const uint32_t* b1, const uint32_t* b2,
                                   uint64_t n, uint32_t* reports, CuckooParScratch& sc, cudaStream_t s);

}  // namespace xpir
