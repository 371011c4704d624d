/* xpir.h — C-ABI of the B200-native Talek server hot path (arXiv 2001.08250).
 *
 * Drop-in boundary for the reference's PIR-server / cuckoo-table / interest-
 * window interfaces (/root/reference/proj/include/oblog/{pir,cuckoo,notify,
 * server}.hpp). Plain pointers and sizes only; no torch or CUDA types in the
 * signatures (streams are passed as `void*` = cudaStream_t, NULL = the
 * library's own stream). Every entry point returns an int status:
 *
 *     XPIR_OK (0)            success
 *     XPIR_EINVAL (-1)       the reference would throw std::invalid_argument
 *     XPIR_ECUDA (-2)        CUDA runtime / kernel error
 *     XPIR_ENOMEM (-3)       device allocation failed
 *     XPIR_ESTATE (-4)       internal invariant (e.g. FIFO ring overflow)
 *
 * and xpir_last_error() returns a thread-local message for the last failure.
 * Functions taking host buffers are synchronous and thread-safe (one mutex per
 * handle). *_dev functions take device pointers and enqueue on `stream`; the
 * scan/expand/mask/reduce ones return without synchronising, while
 * xpir_table_insert_batch_dev and xpir_window_absorb_dev synchronise once (the
 * cuckoo walk's resume state and the absorb range check come back to the host).
 * A store's query scratch is per handle: concurrent *_dev scans on ONE store
 * from different streams must be ordered by the caller.
 *
 * Bit and byte layouts are the reference's:
 *   query vector   bit j = q[j/8] >> (j%8) & 1, ceil(N/8) bytes     (pir.hpp:14-28)
 *   snapshot       bucket i at i*S, slot s of bucket i at (i*depth+s)*item
 *                                                          (pir.hpp:32-41, cuckoo.cpp:23-29)
 *   answer         B x S bytes, request-major                (pir.cpp:41-52)
 */
#ifndef XPIR_H
#define XPIR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define XPIR_OK 0
#define XPIR_EINVAL (-1)
#define XPIR_ECUDA (-2)
#define XPIR_ENOMEM (-3)
#define XPIR_ESTATE (-4)

#define XPIR_SEED_LEN 32   /* crypto::SEED_LEN, crypto.hpp:20 */
#define XPIR_PRF_KEY_LEN 16 /* crypto::PRF_KEY_LEN, crypto.hpp:13 */
#define XPIR_MAX_DISPLACEMENTS 500u /* cuckoo::MAX_DISPLACEMENTS, cuckoo.hpp:15 */

const char* xpir_last_error(void);
int xpir_version(void);
/* Number of kernel launches this process has issued through the library. */
uint64_t xpir_launch_count(void);

/* ------------------------------------------------------------------------ */
/* Sealed snapshot shard (pir::Snapshot, pir.hpp:32-41) resident in HBM.     */
/* A store holds buckets [lo, hi) of an N-bucket snapshot; lo and hi must be  */
/* multiples of 8 unless hi == N (whole query bytes per shard).               */
/* ------------------------------------------------------------------------ */
typedef struct xpir_store xpir_store;

int xpir_store_create(int device, uint32_t bucket_count, uint32_t bucket_size, uint32_t lo,
                      uint32_t hi, xpir_store** out);
int xpir_store_destroy(xpir_store* st);
/* Upload (hi-lo)*S bucket-major bytes from host memory. */
int xpir_store_upload(xpir_store* st, const uint8_t* host_buckets, uint64_t epoch);
/* Copy (hi-lo)*S bytes from device memory (same device). */
int xpir_store_upload_dev(xpir_store* st, const void* dev_src, uint64_t epoch, void* stream);
/* Fill the shard with DetRng bytes: ChaCha20(key, nonce) keystream starting at byte
 * offset lo*S — i.e. the shard's window of one Rng::fill(N*S) call (rng.cpp:25-31). */
int xpir_store_fill_keystream(xpir_store* st, const uint8_t key[32], uint64_t nonce,
                              uint64_t epoch, void* stream);
int xpir_store_info(const xpir_store* st, uint32_t* bucket_count, uint32_t* bucket_size,
                    uint32_t* lo, uint32_t* hi, uint64_t* epoch, void** dev_data);
/* Download `len` shard bytes starting at shard byte `offset` (test helper). */
int xpir_store_download(const xpir_store* st, uint64_t offset, uint64_t len, uint8_t* host_out);

/* ------------------------------------------------------------------------ */
/* PIR read scan — pir::answer / answer_batch (pir.cpp:29-52) + mask_answer   */
/* (pir.cpp:65-69) + the server's answer step of answer_share (server.cpp:    */
/* 115-127). Each request's answer is the XOR of the buckets it selects in    */
/* this shard; with mask_seeds != NULL it is further XORed with               */
/* prng_expand(mask_seed_r, S). q_bits must equal bucket_count (pir.cpp:30). */
/* ------------------------------------------------------------------------ */
int xpir_answer_batch(xpir_store* st, const uint8_t* q, uint64_t q_stride, uint32_t q_bits,
                      uint32_t batch, const uint8_t* mask_seeds, uint8_t* out);
/* Seeded requests: q_r = prng_expand(seed_r, ceil(N/8)) expanded on device (K2). */
int xpir_answer_batch_seeded(xpir_store* st, const uint8_t* seeds, uint32_t batch,
                             const uint8_t* mask_seeds, uint8_t* out);

/* Seed-compressed read shares (l-1 of a read's l shares as 32-byte PRG seeds, only
 * the last explicit): request r is a seed when is_seed[r], its vector then being
 * prng_expand(seed, ceil(N/8)) (crypto.cpp:35-45), else an explicit vector.
 * seeds holds the seeded requests' seeds and q (stride q_stride) the explicit
 * requests' vectors, each compacted in request order. out / mask_seeds as above. */
int xpir_answer_batch_mixed(xpir_store* st, uint32_t batch, const uint8_t* is_seed, const uint8_t* seeds,
                            const uint8_t* q, uint64_t q_stride, uint32_t q_bits, const uint8_t* mask_seeds,
                            uint8_t* out);
/* Device-pointer variants. d_q rows hold the FULL ceil(N/8)-byte vector
 * (the shard reads bytes [lo/8, ceil(hi/8))). d_out is batch*S bytes. */
int xpir_answer_batch_dev(xpir_store* st, const uint8_t* d_q, uint64_t q_stride,
                          uint32_t q_bits, uint32_t batch, const uint8_t* d_mask_seeds,
                          uint8_t* d_out, void* stream);
/* Expand seeds on device into the shard's query window only, then scan.
 * d_qbuf: scratch of batch * xpir_query_window_bytes(st) bytes (or NULL to use an
 * internal buffer). */
int xpir_answer_batch_seeded_dev(xpir_store* st, const uint8_t* d_seeds, uint32_t batch,
                                 const uint8_t* d_mask_seeds, uint8_t* d_out, void* stream);
uint64_t xpir_query_window_bytes(const xpir_store* st);

/* Sharded scan with the cross-GPU XOR reduction FUSED into the scan kernel:
 * rank k owns answer rows [row_bounds[k], row_bounds[k+1]) in its buffer
 * out_ptrs[k] (a local or CUDA-IPC-mapped peer pointer; every buffer holds all B
 * rows at the same offsets); this call is rank self_rank. Inside the kernel the
 * segment partials of each (request tile, 32-byte column tile) accumulate in a
 * local buffer, and the tile's last segment pushes its finished rows to their
 * owners with 64-bit system-scope XOR reductions (NVLink) while other tiles are
 * still scanning: B*S bytes per rank per batch, (G-1)/G of them to peers — the
 * volume of a reduce-scatter. Each owner must have initialised its rows (zero or
 * mask pad, xpir_init_rows_dev) before any rank launches; once every rank's scan
 * has completed the owner's rows are final. Needs S % 32 == 0 and B >= 2048
 * (runs the quad-table M4RM kernel 8); 1..8 ranks. pir::reconstruct semantics. */
int xpir_answer_batch_seeded_peer_dev(xpir_store* st, const uint8_t* d_seeds, uint32_t batch,
                                      uint8_t* const* out_ptrs, const uint32_t* row_bounds, uint32_t n_ranks,
                                      uint32_t self_rank, void* stream);
/* Debug counters of the fused epilogue on this store: bytes pushed to peer ranks'
 * rows and to this rank's own rows since the last reset (synchronises the device). */
int xpir_store_peer_stats(xpir_store* st, uint64_t* remote_bytes, uint64_t* own_bytes, int reset);
/* d_out rows [r0, r1) of S bytes = mask pad prng_expand(mask_seed_r, S) (or zero). */
int xpir_init_rows_dev(int device, uint8_t* d_out, uint32_t r0, uint32_t r1, uint32_t S,
                       const uint8_t* d_mask_seeds, void* stream);

/* K2 alone: d_q[r*q_stride + k] = prng_expand(seed_r)[byte_lo + k], k < nbytes. */
int xpir_expand_queries_dev(int device, const uint8_t* d_seeds, uint32_t batch, uint64_t byte_lo,
                            uint64_t nbytes, uint8_t* d_q, uint64_t q_stride, void* stream);
/* pir::mask_answer (pir.cpp:65-69) for one host answer: out = ans ^ prng_expand(seed, len),
 * the pad generated and applied on device. */
int xpir_mask_answer(const uint8_t* ans, uint64_t len, const uint8_t seed[32], uint8_t* out);
/* K3 alone: d_out[r*S..] ^= prng_expand(mask_seed_r, S). */
int xpir_mask_dev(int device, uint8_t* d_out, const uint8_t* d_mask_seeds, uint32_t batch,
                  uint32_t S, void* stream);
/* K4: d_dst ^= XOR_k d_srcs[k] over `bytes` bytes; sources may be peer pointers
 * (P2P over NVLink) — pir::reconstruct / combine_masked (pir.cpp:54-73). */
int xpir_xor_reduce_dev(int device, uint8_t* d_dst, const uint8_t* const* d_srcs, uint32_t nsrc,
                        uint64_t bytes, void* stream);

/* Scan-kernel tuning / introspection. */
typedef struct {
    int kernel;        /* 0 = auto, 1 = direct select-XOR, 2 = M4RM byte tables (auto variant),
                          4 = M4RM register accumulators, 5 = M4RM half-TMEM accumulators,
                          7 = M4RM nibble tables,
                          8 = M4RM 9-bucket tables, four interleaved per 32-byte column,
                              full-TMEM accumulators (auto for B = 4096 and >= 8192,
                              S % 32 == 0),
                          9 = M4RM 6-bucket tables (64 rows per 6 buckets) */
    int ctas_per_sm;   /* 0 = auto */
    int reserved[6];
} xpir_scan_opts;
int xpir_set_scan_opts(const xpir_scan_opts* o);
/* How host threads wait for the device in this process (all devices): 0 = the
   CUDA runtime's default (spin while there are more cores than contexts),
   1 = spin, 2 = yield, 3 = blocking (threads sleep on an OS primitive). The
   environment variable XPIR_SYNC = spin | yield | blocking sets it at the
   library's first device call. Measured through the reference drop-ins
   (profiles/r02_production_path.jsonl): blocking cuts the real-time cluster's
   mean delivery latency (acceptance criterion 5's replay) from 776 to 590-611 ms
   but makes every synchronous write 4-6x slower (ServerCore::apply_write
   41 -> 178-267 us), so the default stays the runtime's. */
int xpir_set_host_sync(int mode);
/* Which kernel the last scan used (the ids above; 3 = byte-granular, 5 = M4RM half-TMEM). */
int xpir_last_scan_kernel(void);
/* When enabled, CUDA events bracket every scan-kernel launch on its own stream;
 * collect returns the summed kernel milliseconds and launch count since the last
 * collect (synchronising on the recorded events). */
int xpir_scan_timing(int enable);
int xpir_scan_timing_collect(double* total_ms, uint32_t* launches);
/* Microbenchmarks of the two ALU-side ceilings of the scan, measured on `device`:
 * 32-bit LOP3 (acc ^= w & m) lane-ops per second, and LDS.128 shared-memory bytes
 * per second, both chip-wide. */
int xpir_measure_peaks(int device, double* lop3_per_s, double* smem_bytes_per_s,
                       double* sm_clock_mhz);
/* tcgen05.ld (TMEM -> registers) bytes per SM clock with warp-uniform random
 * columns; variant 0..4 = {x1, 4 warps}, {x1, 16}, {x2, 16}, {x4, 16}, {x4, 8}. */
int xpir_probe_tmem(int device, int variant, double* bytes_per_clk_sm);

/* ------------------------------------------------------------------------ */
/* Read batcher ("Read requests are batched and forwarded to   */
/* the GPU"): concurrent single-request callers — server::answer_share       */
/* (server.cpp:115-135) from node.cpp's session/link threads — are coalesced  */
/* into one scan. A batch is sealed at once while the device is idle, else  */
/* when it holds max_batch requests or max_wait_us after its first request; */
/* three pinned batches rotate (one forming, one scanning, one completing). */
/* Callers pack their own query and unpack their own answer. Thread-safe;   */
/* the store must outlive the batcher.                                      */
/* ------------------------------------------------------------------------ */
typedef struct xpir_batcher xpir_batcher;

int xpir_batcher_create(xpir_store* st, uint32_t max_batch, uint32_t max_wait_us, xpir_batcher** out);
/* A batcher with no default store, for snapshots of N buckets x S bytes on
 * `device`: every request names its store (xpir_batcher_answer_on). Batches are
 * sealed adaptively: at once while no batch is in flight, else when full or
 * max_wait_us after their first request, whichever comes first. */
int xpir_batcher_create_geometry(int device, uint32_t N, uint32_t S, uint32_t max_batch, uint32_t max_wait_us,
                                 xpir_batcher** out);
/* Waits for the requests already submitted, then stops the worker. */
int xpir_batcher_destroy(xpir_batcher* b);
/* Blocking: out (bucket_size bytes) = pir::answer(snapshot, q) (pir.cpp:29-39), or
 * pir::mask_answer(pir::answer(snapshot, q), mask_seed) when mask_seed != NULL
 * (answer_share, server.cpp:122-123). q holds ceil(N/8) bytes; q_bits must be N. */
int xpir_batcher_answer(xpir_batcher* b, const uint8_t* q, uint32_t q_bits, const uint8_t* mask_seed,
                        uint8_t* out);
/* The same against another store of the batcher's geometry (whole snapshot, same
 * N and bucket size, same device) — e.g. another sealed epoch of a server ring:
 * requests are batched per (store, masked). The store must stay alive (and, for
 * a server ring image, pinned: xpir_server_snapshot_acquire) until the call
 * returns. */
int xpir_batcher_answer_on(xpir_batcher* b, xpir_store* st, const uint8_t* q, uint32_t q_bits,
                           const uint8_t* mask_seed, uint8_t* out);
int xpir_batcher_stats(xpir_batcher* b, uint64_t* requests, uint64_t* batches, uint64_t* max_batch_seen);

/* ------------------------------------------------------------------------ */
/* Intra-box peer memory for the sharded reduce (CUDA IPC over NVLink).       */
/* ------------------------------------------------------------------------ */
#define XPIR_IPC_HANDLE_BYTES 64
/* Whole device allocations (IPC handles map allocation bases, so buffers shared
 * with peers are allocated here rather than sub-allocated by a caching allocator). */
int xpir_dev_alloc(int device, uint64_t bytes, void** d_ptr);
int xpir_dev_free(int device, void* d_ptr);
int xpir_ipc_get_handle(int device, const void* d_ptr, uint8_t handle[64]);
/* Map a peer process's allocation; enables peer access (NVLink) lazily. */
int xpir_ipc_open(int device, const uint8_t handle[64], void** d_ptr);
int xpir_ipc_close(int device, void* d_ptr);
int xpir_device_sync(int device);

/* ------------------------------------------------------------------------ */
/* Primitives on device, host buffers (parity tests and input generation).    */
/* ------------------------------------------------------------------------ */
/* crypto::prng_expand (crypto.cpp:35-45) */
int xpir_prng_expand(const uint8_t seed[32], uint8_t* out, uint64_t len);
/* DetRng::fill (rng.cpp:25-31): ChaCha20(key, nonce=LE64(nonce)) from block 0. */
int xpir_keystream_dev(int device, const uint8_t key[32], uint64_t nonce, uint64_t byte_offset,
                       uint8_t* d_out, uint64_t len, void* stream);
/* Many fills, one per row: d_out[r*row_stride..+len] = ChaCha20(key, nonce0+r). */
int xpir_keystream_rows_dev(int device, const uint8_t key[32], uint64_t nonce0, uint32_t rows,
                            uint64_t len, uint8_t* d_out, uint64_t row_stride, void* stream);
/* crypto::prf (crypto.cpp:17-33) for n inputs. */
int xpir_prf_batch(const uint8_t key[16], const uint64_t* inputs, uint64_t n, uint64_t modulus,
                   uint64_t* out);
/* Same on device buffers; d_out32 (optional) receives the values as uint32 (bucket indices). */
int xpir_prf_batch_dev(int device, const uint8_t key[16], const uint64_t* d_inputs, uint64_t n,
                       uint64_t modulus, uint64_t* d_out, uint32_t* d_out32, void* stream);
/* The two bucket choices of a write batch in one kernel: beta1 = prf(k1, key, buckets),
 * beta2 = prf(k2, key, buckets) (logproto.cpp:74-75 over crypto::prf). */
int xpir_write_betas_dev(int device, const uint8_t k1[16], const uint8_t k2[16], const uint64_t* d_keys, uint64_t n,
                         uint32_t buckets, uint32_t* d_beta1, uint32_t* d_beta2, void* stream);
/* notify::make_interest (notify.cpp:30-35): out[i*h + k] */
int xpir_make_interest_batch(uint32_t m_bits, uint32_t h, const uint8_t id[16],
                             const uint64_t* seqs, uint64_t n, uint32_t* out);
/* crypto::bloom_positions for one arbitrary item (crypto.cpp:146-166). */
int xpir_bloom_positions(const uint8_t* item, uint64_t len, uint32_t h, uint32_t m_bits,
                         uint32_t* out);
/* crypto::digest = BLAKE2b (crypto.cpp:168-175), computed on the host side of the library. */
int xpir_blake2b(const uint8_t* data, uint64_t len, uint32_t outlen, uint8_t* out);

/* ------------------------------------------------------------------------ */
/* Blocked cuckoo table — cuckoo::Table (cuckoo.hpp:37-84, cuckoo.cpp).       */
/* ------------------------------------------------------------------------ */
typedef struct xpir_table xpir_table;

int xpir_table_create(int device, uint32_t buckets, uint32_t depth, uint64_t capacity,
                      uint64_t item_size, const uint8_t seed[32], xpir_table** out);
int xpir_table_destroy(xpir_table* t);
/* Table::insert (cuckoo.cpp:56-126) for n items in order; reports[4*i..] =
 * {stored, dropped, gc_evicted, displacements} (InsertReport, cuckoo.hpp:23-28). */
int xpir_table_insert_batch(xpir_table* t, const uint32_t* beta1, const uint32_t* beta2,
                            const uint8_t* payload, uint64_t n, uint32_t* reports);
/* Device-resident inputs. beta1/beta2 are range-checked on the device before
 * the walk (one small kernel + a 4-byte read back): the items before the first
 * out-of-range index are inserted, then XPIR_EINVAL (cuckoo.cpp:57-58), exactly
 * as the host entry point and a loop of Table::insert calls. */
int xpir_table_insert_batch_dev(xpir_table* t, const uint32_t* d_beta1, const uint32_t* d_beta2,
                                const uint8_t* d_payload, uint64_t n, uint32_t* d_reports,
                                void* stream);
/* The same batch as a pure stream sequence (no host round trip, no allocation:
 * prefix_done, a cudaEvent_t or NULL, is recorded after the parallel-prefix
 * kernel — a grid-synchronised cooperative launch, so independent bulk work
 * such as the round's interest update is best started after it;
 * capturable in a CUDA graph, e.g. a server's whole write round): the parallel
 * eviction-free prefix, the eviction walk from where it stops, and the payload
 * moves, all reading and advancing the device copy of the table state. Requires
 * xpir_table_reserve(t, >= n) at start-up. xpir_table_finish (after the stream
 * work, outside any capture) reconciles the host mirror, completes what could
 * not run on device (a walk that ran out of staged draws, a batch that moved more
 * slots than the staging holds), and returns XPIR_EINVAL for a bucket index out
 * of range (*n_applied = the inserts before it, as insert_batch_dev). It waits
 * for `stream`: a graph holding the batch must be replayed on that stream (or
 * the caller synchronises before finish). */
int xpir_table_insert_batch_async(xpir_table* t, const uint32_t* d_beta1, const uint32_t* d_beta2,
                                  const uint8_t* d_payload, uint64_t n, uint32_t* d_reports, void* stream,
                                  void* prefix_done);
int xpir_table_finish(xpir_table* t, uint64_t* n_applied);
/* Bucket-range payload shards (the payload scatter goes to the GPU
 * owning each bucket range). A shard table keeps the whole metadata (the walk
 * is replicated: every shard runs the same insert_walk) and the payloads of
 * buckets [lo, hi) only. A round is: insert_walk on every shard; apply_gather on
 * every shard (it reads the pre-round payloads that move into its range, from
 * whichever shard holds them — map.data may be CUDA-IPC peer pointers); a
 * barrier; apply_scatter on every shard (every shard gets all n payloads).
 * xpir_table_insert_batch[_dev] = the three steps on an unsharded table. */
typedef struct {
    uint32_t n;              /* shards, 1..8 */
    uint32_t bucket_lo[9];   /* shard g holds buckets [bucket_lo[g], bucket_lo[g+1]) */
    const uint8_t* data[8];  /* shard g's payload array (xpir_table_device_data) */
} xpir_shard_map;
int xpir_table_create_shard(int device, uint32_t buckets, uint32_t depth, uint64_t capacity, uint64_t item_size,
                            const uint8_t seed[32], uint32_t lo, uint32_t hi, xpir_table** out);
int xpir_table_shard(const xpir_table* t, uint32_t* lo, uint32_t* hi);
/* Range-checked like insert_batch_dev: on XPIR_EINVAL the valid prefix has been
 * walked and the caller still runs apply_gather / apply_scatter for it. */
int xpir_table_insert_walk_dev(xpir_table* t, const uint32_t* d_beta1, const uint32_t* d_beta2, uint64_t n,
                               uint32_t* d_reports, void* stream);
int xpir_table_apply_gather_dev(xpir_table* t, const xpir_shard_map* map, void* stream);
int xpir_table_apply_scatter_dev(xpir_table* t, const uint8_t* d_payload, void* stream);
/* Pre-size the per-round scratch (claim sort buffers, payload staging) for
 * batches of up to max_batch writes, so no allocation happens inside a round. */
int xpir_table_reserve(xpir_table* t, uint64_t max_batch);
/* Table::snapshot bytes (cuckoo.cpp:128-135); of a payload shard: its buckets only. */
int xpir_table_snapshot(const xpir_table* t, uint8_t* host_out);
/* Seal into a store covering the whole table or a bucket range of it (device copy). */
int xpir_table_seal(const xpir_table* t, xpir_store* st, uint64_t epoch, void* stream);
int xpir_table_meta(const xpir_table* t, uint8_t* used, uint32_t* beta1, uint32_t* beta2,
                    uint64_t* stamp);
int xpir_table_counters(const xpir_table* t, uint64_t* writes, uint64_t* live,
                        uint64_t* next_stamp);
/* Table::state_digest (cuckoo.cpp:137-149); whole tables only. */
int xpir_table_state_digest(const xpir_table* t, uint8_t out[32]);
/* Table::slot_used (cuckoo.cpp:160-163). */
int xpir_table_slot_used(const xpir_table* t, uint32_t bucket, uint32_t slot);
void* xpir_table_device_data(const xpir_table* t);

/* ------------------------------------------------------------------------ */
/* Interest window — notify::Window (notify.hpp:57-88, notify.cpp:54-117).    */
/* ------------------------------------------------------------------------ */
typedef struct xpir_window xpir_window;

int xpir_window_create(int device, uint32_t m_bits, uint32_t h, uint32_t w, xpir_window** out);
int xpir_window_destroy(xpir_window* win);
/* Window::absorb: OR positions into the newest delta; EINVAL if any >= m_bits. */
int xpir_window_absorb(xpir_window* win, const uint32_t* positions, uint64_t n);
int xpir_window_absorb_dev(xpir_window* win, const uint32_t* d_positions, uint64_t n,
                           void* stream);
/* Fused make_interest(bp, id, seq_i) + absorb for n writes (BLAKE2b on device). */
int xpir_window_absorb_interest(xpir_window* win, const uint8_t id[16], const uint64_t* seqs,
                                uint64_t n);
int xpir_window_absorb_interest_dev(xpir_window* win, const uint8_t id[16], const uint64_t* d_seqs,
                                    uint64_t n, void* stream);
int xpir_window_rotate(xpir_window* win);
int xpir_window_info(const xpir_window* win, uint64_t* size, uint64_t* base);
int xpir_window_delta(const xpir_window* win, uint64_t i, uint64_t* out_words);
/* Window::digest (notify.cpp:90-107). */
int xpir_window_digest(const xpir_window* win, uint8_t out[32]);
/* Window::digest(count) over the oldest `count` deltas (notify.cpp:92-107). */
int xpir_window_digest_n(const xpir_window* win, uint64_t count, uint8_t out[32]);
/* notify::encode_delta (notify.cpp:139-157) of delta i (0 = oldest), encoded on
 * device: varint(m) || varint(ones) || varint(first position) || varint(gaps).
 * out == NULL: *len = size only. EINVAL when cap < *len. */
int xpir_window_encode_delta(xpir_window* win, uint64_t i, uint8_t* out, uint64_t cap, uint64_t* len);
/* The same from device buffers: d_words holds ceil(m_bits/64) LE words; d_out may
 * be NULL (size query). */
int xpir_encode_delta_dev(int device, const uint64_t* d_words, uint32_t m_bits, uint8_t* d_out, uint64_t cap,
                          uint64_t* len, void* stream);
/* The write's interest field (wire.cpp:154-169, INTEREST_FIELD_LEN = 64 bytes):
 * notify::encode_positions (notify.cpp:182-196) of n writes x h positions into
 * cap-byte fields (d_ok[i] = 0 where the reference throws: the encoding is longer
 * than cap — at m = 2^20, h = 23 about a fifth are), and notify::decode_positions
 * (notify.cpp:198-214): d_count[i] = count, positions in d_pos[i*cap ...], or
 * 0xffffffff for std::nullopt. h <= 128, cap <= 4096. */
int xpir_encode_positions_dev(int device, const uint32_t* d_pos, uint32_t h, uint64_t n, uint32_t cap,
                              uint8_t* d_fields, uint8_t* d_ok, void* stream);
int xpir_decode_positions_dev(int device, const uint8_t* d_fields, uint32_t cap, uint64_t n, uint32_t* d_pos,
                              uint32_t* d_count, void* stream);
/* notify::decode_delta (notify.cpp:159-180), decoded on device. XPIR_EINVAL is the
 * reference's std::nullopt (malformed input). words == NULL: header only
 * (*m_bits); else words receives ceil(m/64) words (EINVAL if words_cap is short). */
int xpir_decode_delta(int device, const uint8_t* buf, uint64_t len, uint32_t* m_bits, uint64_t* words,
                      uint64_t words_cap);

/* ------------------------------------------------------------------------ */
/* Replica state machine — server::ServerCore (server.hpp:57-98,             */
/* server.cpp:28-91) on device: cuckoo table + interest window + a ring of     */
/* at most epoch_ring sealed stores. Creation rotates the window once and     */
/* seals epoch 1 (server.cpp:40-42). A sealed store is re-sealed incrementally */
/* when it falls off the ring: only slots rewritten since it was last synced  */
/* are copied (the reference copies the whole table per seal).               */
/* ------------------------------------------------------------------------ */
typedef struct xpir_server xpir_server;

int xpir_server_create(int device, uint32_t buckets, uint32_t depth, uint64_t capacity, uint64_t item_size,
                       const uint8_t seed[32], uint32_t m_bits, uint32_t h, uint32_t window_deltas,
                       uint32_t rotate_writes, uint32_t epoch_ring, xpir_server** out);
/* A server whose table and sealed stores hold the payloads of buckets [lo, hi)
 * (one rank of a bucket-range sharded deployment; the walk, the interest window
 * and the epoch numbering are replicated on every rank). */
int xpir_server_create_shard(int device, uint32_t buckets, uint32_t depth, uint64_t capacity, uint64_t item_size,
                             const uint8_t seed[32], uint32_t m_bits, uint32_t h, uint32_t window_deltas,
                             uint32_t rotate_writes, uint32_t epoch_ring, uint32_t lo, uint32_t hi,
                             xpir_server** out);
int xpir_server_destroy(xpir_server* sv);
/* n calls of ServerCore::apply_write (server.cpp:58-73) in order — insert,
 * absorb the write's h_per_write interest positions, rotate every rotate_writes
 * writes — then seal once if seal_after (the last write's seal_after). */
int xpir_server_apply_round(xpir_server* sv, const uint32_t* beta1, const uint32_t* beta2, const uint8_t* payload,
                            const uint32_t* interest, uint32_t h_per_write, uint64_t n, int seal_after,
                            uint32_t* reports, uint64_t* sealed_epoch);
/* apply_round on one rank of a sharded deployment: every rank calls it with the
 * same writes; barrier(ctx) must return once every rank has reached it (between
 * the payload gather and scatter phases, see xpir_table_apply_gather_dev). */
int xpir_server_apply_round_sharded(xpir_server* sv, const uint32_t* beta1, const uint32_t* beta2,
                                    const uint8_t* payload, const uint32_t* interest, uint32_t h_per_write,
                                    uint64_t n, int seal_after, const xpir_shard_map* map,
                                    void (*barrier)(void*), void* barrier_ctx, uint32_t* reports,
                                    uint64_t* sealed_epoch);
/* Server start-up: size the per-round scratch for rounds of up to max_batch
 * writes and allocate every sealed image of the ring up front, so a round never
 * allocates device memory. */
int xpir_server_reserve(xpir_server* sv, uint64_t max_batch);
int xpir_server_seal(xpir_server* sv, uint64_t* epoch);            /* seal_epoch, server.cpp:75-81 */
/* snapshot_at (server.cpp:83-87); epoch 0 = latest. The store stays owned by the
 * server and valid until its epoch leaves the ring. */
int xpir_server_snapshot(xpir_server* sv, uint64_t epoch, xpir_store** st);
/* snapshot_at with a reader pin (the reference keeps a retired snapshot alive
 * through its shared_ptr, server.cpp:83-87): the image is not reused while
 * pinned — a seal that pushes a pinned epoch off the ring retires it and seals
 * into another image; the last release returns it to the spare pool.
 * epoch 0 = latest; *epoch_out (optional) = the epoch pinned. */
int xpir_server_snapshot_acquire(xpir_server* sv, uint64_t epoch, xpir_store** st, uint64_t* epoch_out);
int xpir_server_snapshot_release(xpir_server* sv, xpir_store* st);
/* ServerCore::make_freeze (server.cpp:45-56): base, newest (= window newest - 1),
 * digest over the frozen deltas and their count; their wire bytes are
 * xpir_window_encode_delta(window, k, ...) for k < count. */
int xpir_server_freeze(xpir_server* sv, uint64_t* base, uint64_t* newest, uint8_t digest[32], uint64_t* count);
int xpir_server_info(xpir_server* sv, uint64_t* writes, uint64_t* latest_epoch, uint64_t* oldest_epoch,
                     xpir_table** table, xpir_window** window);

#ifdef __cplusplus
}
#endif
#endif
