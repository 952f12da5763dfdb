/*
 * fsx.h -- C ABI of the B200-native sidecar data plane (libfsx.so).
 *
 * Drop-in boundary for the reference's sidecar hot path (fissim,
 * /root/reference/proj/include/fissim/sidecar.hpp).  The reference is
 * header-only C++ with no FFI of its own; these are the entry points its
 * C++ SidecarFabric would bind to move bytes on B200s.  Every
 * function cites the reference interface it replaces as file:line relative to
 * /root/reference/proj.  The C++ SidecarFabric-compatible engine
 * (include/fsx/fabric.hpp) and the Python bindings sit on top of this header.
 *
 * Conventions
 *  - All functions return int status: 0 = OK, otherwise 1 + the ordinal of
 *    fissim::ErrorCode (include/fissim/common.hpp:29-47); the message is in
 *    fsx_last_error() (thread-local).  The C++ shim rethrows fissim::Error.
 *  - "gpu" is the fabric's logical GPU id (the keys of the reference's
 *    gpu_to_node map, sidecar.hpp:242-248).  Each logical GPU is bound to a
 *    CUDA device ordinal at fsx_open().
 *  - Pointers named d_* are device pointers, h_* host pointers.  `stream` is a
 *    cudaStream_t passed as void* (NULL = the fabric's own stream for that
 *    device).  Calls that take a stream are asynchronous on it.
 *  - There is NO CPU fallback: without a CUDA device fsx_open fails with
 *    FSX_E_CONFIG and every data-moving call fails.
 */
#ifndef FSX_H
#define FSX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: 1 + fissim::ErrorCode ordinal (common.hpp:29-47) ---- */
#define FSX_OK 0
#define FSX_E_VALIDATION 1
#define FSX_E_NOT_FOUND 3
#define FSX_E_OOM 5
#define FSX_E_INTEGRITY 10
#define FSX_E_PROTOCOL 11
#define FSX_E_TIMEOUT 12
#define FSX_E_CONFIG 14
#define FSX_E_CANCELLED 16
#define FSX_E_INTERNAL 17

/* Transport, sidecar.hpp:32 (enum class Transport { LocalBuffer, NetworkStream }) */
#define FSX_TRANSPORT_LOCAL_BUFFER 0
#define FSX_TRANSPORT_NETWORK_STREAM 1

typedef struct fsx_fabric fsx_fabric;

/* Thread-local message of the last failing call on this thread. */
const char* fsx_last_error(void);
/* Library version string and the CUDA arch it was built for. */
const char* fsx_version(void);
/* Number of visible CUDA devices (0 on a GPU-less host; never a fallback). */
int fsx_device_count(int* n);
/* sizeof of the ABI structs (fsx_merge_batch, fsx_transfer, fsx_stats), so
 * bindings can check their layouts without a GPU. */
int fsx_abi_sizes(int32_t* merge_batch, int32_t* transfer, int32_t* stats);

/* ---- fabric lifetime ------------------------------------------------------
 * Replaces SidecarFabric(SimKernel&, std::map<int,int> gpu_to_node, SidecarConfig)
 * (sidecar.hpp:242-248).  gpu_ids[i] lives on node node_ids[i] and is bound to
 * CUDA device devices[i] (devices == NULL or devices[i] < 0 -> gpu_id % count).
 * Peer access is enabled between every pair of distinct bound devices. */
int fsx_open(int n_gpus, const int* gpu_ids, const int* node_ids, const int* devices,
             fsx_fabric** out);
int fsx_close(fsx_fabric* f);

/* SidecarFabric::node_of (sidecar.hpp:255-260): FSX_E_NOT_FOUND for an unknown gpu. */
int fsx_node_of(fsx_fabric* f, int gpu, int* node);
/* SidecarFabric::route (sidecar.hpp:250-253). */
int fsx_route(fsx_fabric* f, int src_gpu, int dst_gpu, int* transport);
/* CUDA device ordinal bound to a logical gpu. */
int fsx_device_of(fsx_fabric* f, int gpu, int* device);

/* ---- receive slabs --------------------------------------------------------
 * The reference keeps one shm NodeArena per node (sidecar.hpp:106-135,
 * 244-247).  Here every consumer GPU owns a device-memory receive slab with the
 * same allocation policy: first fit in offset order, 64 B alignment, zero-byte
 * requests take one 64 B unit, coalescing free (sidecar.hpp:149-186). */
int fsx_slab_register(fsx_fabric* f, int gpu, int64_t bytes);
/* NodeArena::alloc (sidecar.hpp:149-163).  *off = -1 when nothing fits (the
 * caller backlogs, sidecar.hpp:329-334); that is not an error. */
int fsx_slab_alloc(fsx_fabric* f, int gpu, int64_t len, int64_t* off);
/* NodeArena::free_seg (sidecar.hpp:165-186): FSX_E_INTERNAL on double free. */
int fsx_slab_free(fsx_fabric* f, int gpu, int64_t off);
/* Batch forms for a whole request batch (one call instead of one per item):
 * alloc_n is all-or-nothing (offs[i] = -1 for every i when the batch does not
 * fit, nothing held); free_n frees every offset (FSX_E_INTERNAL on the first
 * double free, after freeing the rest). */
int fsx_slab_alloc_n(fsx_fabric* f, int gpu, int32_t n, const int64_t* lens, int64_t* offs);
int fsx_slab_free_n(fsx_fabric* f, int gpu, int32_t n, const int64_t* offs);
/* NodeArena::data (sidecar.hpp:188), as a device pointer into the slab. */
int fsx_slab_ptr(fsx_fabric* f, int gpu, int64_t off, void** d_ptr);
/* NodeArena::segments_in_use / bytes_in_use / peak_bytes / capacity
 * (sidecar.hpp:147, 190-192). */
int fsx_slab_usage(fsx_fabric* f, int gpu, int64_t* segments, int64_t* bytes_in_use,
                   int64_t* peak_bytes, int64_t* capacity);
/* Copy n bytes of a slab segment into host memory and wait for them: the
 * owned-vector delivery of the reference ChunkCallback path
 * (sidecar.hpp:543-544).  Zero-copy consumers use fsx_slab_ptr instead. */
int fsx_slab_read(fsx_fabric* f, int gpu, int64_t off, void* h_dst, int64_t n, void* stream);
/* Host -> slab copy of n bytes at off, waited for: the producer half of the
 * multi-process boundary, where a worker stages its payload in its own
 * exported outbox slab instead of copying it into a TCP frame
 * (executor_worker.hpp:245-256). */
int fsx_slab_write(fsx_fabric* f, int gpu, int64_t off, const void* h_src, int64_t n, void* stream);
/* Cross-process slabs (executor_worker.hpp:63-87 shm-name handshake ->
 * cudaIpcMemHandle).  export writes 64 handle bytes; import maps a slab owned
 * by another process as logical `gpu` (chunk flags included). */
int fsx_slab_export(fsx_fabric* f, int gpu, void* handle64, int64_t* bytes);
int fsx_slab_import(fsx_fabric* f, int gpu, const void* handle64, int64_t bytes);
/* Raw CUDA IPC mapping of memory exported by another process (a worker's
 * outbox slab, fsx_slab_export there), opened on `gpu`'s device; replaces the
 * worker-side MappedArena shm_open/mmap (executor_worker.hpp:210-227) on the
 * parent side.  fsx_close() closes mappings still open. */
int fsx_ipc_open(fsx_fabric* f, int gpu, const void* handle64, void** d_ptr);
int fsx_ipc_close(fsx_fabric* f, void* d_ptr);

/* ---- chunk flags ----------------------------------------------------------
 * Per-consumer-GPU ring of 64-bit completion flags, mirrored in device memory
 * (for consumer kernels that start early) and in mapped pinned host memory
 * (for the host progress thread).  A flag holds the token of the transfer
 * chunk that last completed there; tokens are unique per fsx_forward call, so
 * slots never need resetting. */
int fsx_flags_alloc(fsx_fabric* f, int dst_gpu, int32_t n, int64_t* flag_base);
int fsx_flag_ptr(fsx_fabric* f, int dst_gpu, int64_t flag_idx, uint64_t** d_flag);

/* ---- forwarding (K1) --------------------------------------------------------
 * Replaces the payload placement of SidecarFabric::send / try_place_local
 * (sidecar.hpp:302-347, 465-483: checksum + copy into PendingSend + memcpy into
 * the arena).  An sm_100a kernel on src_gpu's device pushes `bytes` from d_src
 * into dst_gpu's slab at dst_off with 16-byte stores (NVLink/NVSwitch P2P when
 * the devices differ, HBM copy when they are the same), chunk by chunk; when
 * chunk c is fully stored its flag flag_base + c is set to the token
 * (release, system scope).  n_chunks = ceil(bytes / chunk_bytes) (1 when
 * chunk_bytes <= 0 or >= bytes); chunk_bytes must be a multiple of 16.
 * token is in/out: a non-zero *token on entry is used as given (tokens agreed
 * out of band, e.g. across processes); otherwise a fresh one is drawn. */
int fsx_forward(fsx_fabric* f, int src_gpu, const void* d_src, int dst_gpu, int64_t dst_off,
                int64_t bytes, int64_t chunk_bytes, int64_t flag_base, uint64_t* token,
                void* stream);
/* fsx_forward with options.  FSX_FWD_HOST_NOTIFY (set by fsx_forward) also
 * mirrors each chunk flag into mapped host memory for fsx_wait /
 * fsx_chunk_ready; leave it out when only device consumers (a merge with
 * early start, fsx_stream_wait_flags, or plain stream order) wait on the chunks,
 * which saves the posted PCIe store at the kernel tail. */
#define FSX_FWD_HOST_NOTIFY 1u
/* FSX_FWD_L2_KEEP: store the slab bytes with L2 evict_last priority, for a
 * consumer on the same GPU that reads them right after (the merge); the
 * producer's source is always read with evict_first. */
#define FSX_FWD_L2_KEEP 2u
/* FSX_FWD_BULK: move this batch's tiles with the bulk-copy engine
 * (forward_tma_kernel: cp.async.bulk global->shared->global, 32 KiB per
 * 32-thread CTA, 16 registers) instead of register loads/stores -- the faster
 * K1 when it runs alone (1.01 of the measured copy peak on 256 MiB).  Local
 * or peer (NVLink) slabs; it applies when every transfer of the batch is
 * 16-byte aligned without a fused digest, else the register tile kernel runs. */
#define FSX_FWD_BULK 4u
/* FSX_FWD_PEER_GPU_COUNT: for peer (NVLink) destinations, count each tile
 * into its chunk with a gpu-scope acq_rel atomic and let the tile that
 * completes a chunk make the whole chunk visible to the consumer GPU with one
 * fence.sc.sys before the system-scope flag store, instead of a system-scope
 * acq_rel atomic per tile (the default).  No effect on local slabs. */
#define FSX_FWD_PEER_GPU_COUNT 16u
/* FSX_FWD_DMA: move each chunk with the copy engine (cudaMemcpyAsync) and
 * publish the transfer's chunk flags with one tiny flag kernel behind the
 * copies (stream order) instead of launching K1: a small isolated transfer
 * then costs the copy engine's latency plus a one-thread launch (1.7-1.8 us
 * for 64 KiB-1 MiB) instead of K1's tiles and per-tile completion protocol
 * (2.6-2.8 us).  A transfer's flags turn together, after its last chunk.
 * Chosen automatically for a batch of at most FSX_FWD_DMA_MAX_CHUNKS chunks (one
 * transfer of one chunk: a memcpy + flag launch per chunk or transfer would
 * cost more than one K1 launch)
 * and FSX_FWD_DMA_MAX_BYTES bytes in total, every destination local, no fused
 * digest and no FSX_FWD_L2_KEEP (FSX_FWD_KERNEL or FSX_FWD_BULK force K1);
 * with FSX_FWD_DMA it applies to any batch, peer destinations included.
 * Ignored (K1 runs) when any transfer asks for a fused digest. */
#define FSX_FWD_DMA 32u
/* FSX_FWD_KERNEL: always the register-tile K1 (no copy-engine form, no
 * automatic bulk-copy tiles).  Without FSX_FWD_KERNEL / FSX_FWD_BULK /
 * FSX_FWD_L2_KEEP, a local batch above 2 MiB that is not taken by the
 * copy-engine form runs the bulk-copy tiles (forward_tma_kernel) when every
 * transfer is 16-byte aligned without a fused digest. */
#define FSX_FWD_KERNEL 64u
#define FSX_FWD_DMA_MAX_CHUNKS 1
#define FSX_FWD_DMA_MAX_BYTES (16ll << 20)
int fsx_forward_ex(fsx_fabric* f, int src_gpu, const void* d_src, int dst_gpu, int64_t dst_off,
                   int64_t bytes, int64_t chunk_bytes, int64_t flag_base, uint64_t* token,
                   uint32_t options, void* stream);
/* Several transfers of one source device in one K1 launch (ExecutorBase::
 * emit_output fans one output out to every dest gpu, executor_sim.hpp:223-226;
 * an encoder batch emits several items at once, :321-336).  token is in/out
 * per transfer as above.  All t[i].src_gpu must be bound to the same device.
 * Up to FSX_FWD_MAX_BATCH transfers go in one launch (kernel parameter
 * space); more take ceil(n / FSX_FWD_MAX_BATCH) launches. */
#define FSX_FWD_MAX_BATCH 64
typedef struct fsx_transfer {
  int32_t src_gpu;
  int32_t dst_gpu;
  const void* d_src;
  int64_t dst_off;
  int64_t bytes;
  int64_t chunk_bytes;
  int64_t flag_base;
  uint64_t token;
  uint64_t* d_digest; /* optional device u64 (zeroed, see fsx_u64_slot): += dg64 of
                         the bytes, fused into K1 (see fsx_digest) */
} fsx_transfer;
int fsx_forward_batch(fsx_fabric* f, int32_t n, fsx_transfer* t, uint32_t options, void* stream);
/* Same contract for a HOST source span (the reference send(span) path,
 * sidecar.hpp:302): host->device copy straight into the consumer slab on
 * dst_gpu's device, then the chunk flags.  Pageable or pinned h_src. */
int fsx_forward_host(fsx_fabric* f, const void* h_src, int dst_gpu, int64_t dst_off,
                     int64_t bytes, int64_t chunk_bytes, int64_t flag_base, uint64_t* token,
                     void* stream);
/* fsx_forward_host that also returns the dg64 of the source bytes as sent:
 * computed in the same pass that stages a pageable source (copy and digest
 * fused on the host copy threads), or alongside the DMA of a pinned one.  The
 * drop-in's host-span sends (sidecar.hpp:302-347) use it for the envelope's
 * checksum. */
int fsx_forward_host_digest(fsx_fabric* f, const void* h_src, int dst_gpu, int64_t dst_off,
                            int64_t bytes, int64_t chunk_bytes, int64_t flag_base, uint64_t* token,
                            void* stream, uint64_t* digest);
/* Non-blocking readiness of one chunk (host mirror of the flag). */
int fsx_chunk_ready(fsx_fabric* f, int dst_gpu, int64_t flag_idx, uint64_t token, int* ready);
/* ---- small host messages ----------------------------------------------------
 * The reference's per-token sends (executor_sim.hpp:540-564: thinker hidden
 * states, talker codes) are 4 B - 7 KiB host spans, each handed to a
 * ChunkCallback as an owned host vector after a checksum (sidecar.hpp:527-563).
 * fsx_put_small copies the span into a slot of a pinned mapped mailbox,
 * publishes a descriptor on the destination device's small-message lane and
 * returns: a one-CTA service kernel on that device (launched on demand, exits
 * after 200 us without work) moves each published message into its slab
 * segment, digests the bytes it read (sent) and the segment read back (landed)
 * and marks it done -- no launch, event or host digest per message.
 * fsx_ticket_wait blocks until the message is served (its bytes are then in
 * the slab) and returns the sent bytes (valid until fsx_ticket_free) and the
 * landed dg64; fsx_ticket_digests returns both digests (sent == landed: the
 * slab holds the bytes as sent).  *ticket = -1 (not an error) when n is 0 or
 * > FSX_SMALL_MAX or the mailbox / lane ring is full: use fsx_forward_host.
 * fsx_flush_small is a no-op kept for callers of the batched form. */
#define FSX_SMALL_MAX 65536
int fsx_put_small(fsx_fabric* f, int dst_gpu, int64_t dst_off, const void* h_src, int64_t n,
                  int64_t* ticket);
/* The same for a DEVICE source (a thinker's hidden-state row on its GPU, this
 * device's memory or a peer's): no host staging, the lane kernel reads the
 * row in place, so the source must stay unchanged until the ticket is served
 * (fsx_ticket_wait).  fsx_ticket_wait returns no host bytes for it
 * (*h_bytes = NULL); fsx_ticket_take copies the landed segment out. */
int fsx_put_small_device(fsx_fabric* f, int dst_gpu, int64_t dst_off, const void* d_src, int64_t n,
                         int64_t* ticket);
/* Allocate the slab segment (NodeArena first fit, as fsx_slab_alloc) and
 * publish the message on the lane in one call: *dst_off = -1 when the slab is
 * full (the reference parks the send, sidecar.hpp:329-334); *ticket = -1 when
 * the lane declines (the segment stays allocated for the caller's own copy). */
int fsx_put_small_alloc(fsx_fabric* f, int dst_gpu, const void* src, int64_t n, int src_is_device,
                        int64_t* dst_off, int64_t* ticket);
int fsx_flush_small(fsx_fabric* f);
int fsx_ticket_wait(fsx_fabric* f, int64_t ticket, const void** h_bytes, uint64_t* digest);
int fsx_ticket_digests(fsx_fabric* f, int64_t ticket, uint64_t* sent, uint64_t* landed);
int fsx_ticket_free(fsx_fabric* f, int64_t ticket);
/* Wait, copy the first n bytes of the message to h_dst (may be NULL), return
 * both digests and free the ticket, in one call (the drop-in's delivery). */
int fsx_ticket_take(fsx_fabric* f, int64_t ticket, void* h_dst, int64_t n, uint64_t* sent,
                    uint64_t* landed);

/* Host wait until flags [flag_base, flag_base + n) all equal token;
 * FSX_E_TIMEOUT after timeout_us (< 0 = forever). */
int fsx_wait(fsx_fabric* f, int dst_gpu, int64_t flag_base, int32_t n, uint64_t token,
             int64_t timeout_us);
/* Device-side wait: enqueue on `stream` (a stream of dst_gpu's device) a tiny
 * kernel that spins on the device flags (acquire, system scope) so that work
 * queued after it starts exactly when the chunks have landed. */
int fsx_stream_wait_flags(fsx_fabric* f, int dst_gpu, int64_t flag_base, int32_t n,
                          uint64_t token, void* stream);
/* Enqueue on `stream` (any device of this process) a store of token into
 * flags [flag_base, flag_base + n) of dst_gpu's slab (release, system scope):
 * the cross-process acknowledgement (ack_raw, sidecar.hpp:287-290) and any
 * consumer->producer signal ride on it. */
int fsx_signal_flags(fsx_fabric* f, int dst_gpu, int64_t flag_base, int32_t n, uint64_t token,
                     int src_gpu, void* stream);

/* ---- merge (K3) -------------------------------------------------------------
 * New on this path: the reference consumer discards the bytes
 * (executor_sim.hpp:382-392).  Contract: request r
 * owns rows [req_row_off[r], req_row_off[r+1]) of d_embeds / d_token_ids and
 * items [req_item_off[r], req_item_off[r+1]) in input-slot order
 * (record_replay.hpp:404-416).  The k-th row of request r whose token id equals
 * placeholder_id receives row k of concat(item rows).  Text rows are never
 * touched.  If the placeholder count of request r differs from the sum of its
 * item rows, request r is left untouched and d_status[r] = FSX_E_VALIDATION
 * (0 otherwise).  Rows are moved as opaque bytes (bf16 NaN/Inf patterns
 * survive).  All arrays are DEVICE arrays on gpu's device.  Optional early
 * start: when d_item_flag is non-NULL, row j of item i is copied only after
 * d_item_flag[i][j / d_item_chunk_rows[i]] == d_item_token[i].
 * Two phases: a placeholder scan (needs only token ids, so it can run while
 * the payload is still in flight) and the row copy.  mode selects both
 * (FULL), the scan alone (SCAN_ONLY) or the copy of an already-scanned batch
 * (COPY_ONLY, same d_scratch / d_status). */
#define FSX_MERGE_FULL 0
#define FSX_MERGE_SCAN_ONLY 1
#define FSX_MERGE_COPY_ONLY 2
/* Option bits OR-ed into `mode` (copy phase, LDG kernel):
 * FSX_MERGE_DISCARD   once a placeholder row has been read from its slab
 *   segment, discard the row's L2 lines (discard.global.L2): a merged slab
 *   segment is dead until it is released and rewritten, so its bytes, which
 *   K1 (or the peer's NVLink stores) left in this GPU's L2, are never written
 *   back to HBM.  The segment must not be read again before it is rewritten.
 * FSX_MERGE_COLOCATED early start while the producer's K1 runs on this same
 *   GPU: at most one merge CTA per SM, so spinning merge warps can never take
 *   every slot K1 needs to make progress.  Without it an early-start merge is
 *   a full grid (warp per row, resident CTAs spin on their chunk flags): for
 *   producers on another GPU or in another process. */
#define FSX_MERGE_DISCARD 0x100
#define FSX_MERGE_COLOCATED 0x200
#define FSX_MERGE_MODE_MASK 0xff
typedef struct fsx_merge_batch {
  int32_t num_requests;
  int32_t num_items;
  int64_t row_bytes;                 /* hidden_dim * embed_elem_bytes (profiles.hpp:278-283) */
  int32_t placeholder_id;
  int32_t mode;                      /* FSX_MERGE_FULL / _SCAN_ONLY / _COPY_ONLY */
  void* d_embeds;                    /* [sum T, row_bytes] */
  const int32_t* d_token_ids;        /* [sum T] */
  const int64_t* d_req_row_off;      /* [R + 1] */
  const int64_t* d_req_item_off;     /* [R + 1] */
  const void* const* d_item_src;     /* [M] device pointers (slab views) */
  const int64_t* d_item_row_off;     /* [M + 1] prefix sums of item rows */
  int32_t* d_scratch;                /* [sum item rows] scratch (the scan's prompt row
                                        per placeholder row; total_rows < 2^31) */
  int32_t* d_status;                 /* [R] out */
  const uint64_t* const* d_item_flag; /* optional [M] */
  const uint64_t* d_item_token;      /* optional [M] */
  const int64_t* d_item_chunk_rows;  /* optional [M] */
  int64_t total_rows;                /* sum T (== d_req_row_off[R]) */
  int64_t total_item_rows;           /* == d_item_row_off[M] */
} fsx_merge_batch;
int fsx_merge(fsx_fabric* f, int gpu, const fsx_merge_batch* b, void* stream);

/* Direct placement: the forward fused with the merge.  Where the reference
 * copies a payload into the consumer's arena (sidecar.hpp:465-483) and the
 * consumer then copies it out (:543-544) -- and here K1 pushes it into a slab
 * that K3 then reads -- the producer writes every item row straight into the
 * consumer's placeholder rows: one K3b launch on src_gpu's device with
 *   d_item_src                      producer buffers (src_gpu memory),
 *   d_embeds, d_scratch, d_status   consumer arrays (dst_gpu memory: the same
 *                                   device, a peer, or IPC-opened),
 * so the payload crosses HBM / NVLink once and no slab segment is held.
 * mode: FSX_MERGE_COPY_ONLY uses the positions and statuses the consumer's scan
 * (fsx_merge FSX_MERGE_SCAN_ONLY on dst_gpu, ordered before this call) left in
 * d_scratch / d_status; FSX_MERGE_FULL scans first.  Rows of requests whose
 * status is not 0 are left untouched, as in fsx_merge.  No early-start or
 * discard bits (FSX_E_VALIDATION).  done_flag >= 0: after the rows have landed,
 * dst_gpu's flag done_flag is set to token (release, system scope), for a
 * consumer in another process (fsx_wait / fsx_stream_wait_flags).
 * Counts as one forward of total_item_rows * row_bytes bytes and one merge. */
int fsx_forward_place(fsx_fabric* f, int src_gpu, int dst_gpu, const fsx_merge_batch* b,
                      int64_t done_flag, uint64_t token, void* stream);

/* The forward and the merge as ONE kernel (the tee).  When the producer's
 * buffers are addressable from one device -- N = 1, producer and consumer on
 * the same GPU -- the slab pass reads every item row once and stores it twice:
 * into the item's slab segment with per-chunk flags, exactly as
 * fsx_forward_batch would (t[i]: dst_gpu, dst_off, chunk_bytes, flag_base,
 * token in/out), and into its placeholder row, exactly as fsx_merge would (b:
 * the consumer's batch, whose d_item_src[i] must be t[i].d_src).  The payload
 * crosses HBM three times instead of four (K1 writes the slab, K3 reads it
 * back), in one launch per 64 items.  n == b->num_items, t[i].bytes == item i's
 * rows * row_bytes, chunk_bytes whole rows (or <= 0: one chunk).  mode:
 * FSX_MERGE_FULL (scan first, same stream) or FSX_MERGE_COPY_ONLY (positions and
 * statuses from an earlier scan); no early-start or discard bits.  Options:
 * FSX_FWD_HOST_NOTIFY, FSX_FWD_L2_KEEP, FSX_FWD_PEER_GPU_COUNT.  Items of a
 * request that failed validation are still forwarded; its prompt rows are
 * left untouched.  Runs on t[0].src_gpu's device; counts as n forwards and
 * one merge. */
int fsx_forward_merge(fsx_fabric* f, int32_t n, fsx_transfer* t, const fsx_merge_batch* b,
                      uint32_t options, void* stream);

/* ---- streaming channels (config C) ------------------------------------------
 * The small-message streams of the reference: thinker hidden states, one
 * [hidden_dim] row per decoded token and request (executor_sim.hpp:556-562),
 * and talker codes, 4 B per chunk (:543-549), each a streaming DataRef sent
 * with seq = token index and delivered strictly in seq order
 * (sidecar.hpp:527-531).  Per-message send()+envelope+event is replaced by one
 * launch per decode step for all active requests: a channel is one stream
 * (one request's streaming ref) with a ring of `slots` rows in the consumer's
 * slab, per-slot flags and device-resident head/tail counters.
 *   push: row i of d_rows (row_stride apart) -> next slot of channels[i]; waits
 *         (in kernel) while the ring is full; flag = tag(seq), release.
 *   pull: for each channels[i], waits for its next seq (acquire), copies it to
 *         row i of d_out and frees the slot (tail = seq + 1).
 * All channels of one push share a source device, of one pull a consumer
 * device.  fsx_channel_progress reads (produced, consumed) for tests. */
int fsx_channel_open(fsx_fabric* f, int src_gpu, int dst_gpu, int64_t row_bytes, int32_t slots,
                     int32_t* channel);
int fsx_channel_close(fsx_fabric* f, int32_t channel);
int fsx_channel_push(fsx_fabric* f, int32_t n, const int32_t* channels, const void* d_rows,
                     int64_t row_stride, void* stream);
int fsx_channel_pull(fsx_fabric* f, int32_t n, const int32_t* channels, void* d_out,
                     int64_t out_stride, void* stream);
/* Several groups of channels in one step -- e.g. a decode step's thinker
 * hidden rows and talker codes, different row sizes from different buffers --
 * moved by one push launch and one pull launch (up to 48 rows per launch)
 * instead of one per group.  Group g: channels[0..n) with rows at
 * d_rows + i * stride (push: the producer rows; pull: the output rows).  Same
 * rules as fsx_channel_push / fsx_channel_pull per row. */
typedef struct fsx_chan_group {
  int32_t n;
  const int32_t* channels;
  void* d_rows;
  int64_t stride;
} fsx_chan_group;
int fsx_channel_push_groups(fsx_fabric* f, int32_t n_groups, const fsx_chan_group* groups,
                            void* stream);
int fsx_channel_pull_groups(fsx_fabric* f, int32_t n_groups, const fsx_chan_group* groups,
                            void* stream);
int fsx_channel_progress(fsx_fabric* f, int32_t channel, uint64_t* produced, uint64_t* consumed);

/* ---- synthesis (K0) ---------------------------------------------------------
 * synth_payload_into (common.hpp:247-259) on the device: byte-identical to the
 * reference stream.  Used by producers/tests/bench to create inputs. */
int fsx_synth_payload(fsx_fabric* f, int gpu, uint64_t seed, void* d_dst, int64_t n,
                      void* stream);

/* ---- integrity digest -------------------------------------
 * checksum64 (common.hpp:221-241) is a serial chain; on the device hop fsx
 * uses dg64, a lane-parallel, position-sensitive digest:
 *   dg64 = n * 0x9e3779b97f4a7c15 + sum_k f(w_k ^ (k + 1) * 0xbf58476d1ce4e5b9) mod 2^64
 *   f(x) = y ^ (y >> 29), y = x * 0x94d049bb133111eb,
 * w_k the k-th little-endian 8-byte word (last one zero-padded).  K1 computes it
 * for free while copying (fsx_transfer.d_digest); fsx_digest recomputes it
 * over any device range (consumer-side verification of a slab segment).
 *   fsx_digest: async, *d_accum += dg64(d_ptr[0..n)) on gpu's device.
 *   fsx_u64_slot: a zeroed device u64 from a per-device ring (zeroed on stream).
 *   fsx_read_u64: synchronous read of a device u64 through `stream`. */
int fsx_digest(fsx_fabric* f, int gpu, const void* d_ptr, int64_t n, uint64_t* d_accum,
               void* stream);
int fsx_u64_slot(fsx_fabric* f, int gpu, uint64_t** d_slot, void* stream);
int fsx_read_u64(fsx_fabric* f, int gpu, const uint64_t* d, uint64_t* h, void* stream);

/* ---- host helpers -----------------------------------------------------------
 * Device ordinal owning p, or -1 for host / unregistered memory (never fails).
 * Lets the send(span) entry point (sidecar.hpp:302) take a producer tensor that
 * already lives on the GPU down the K1 path instead of the host copy path. */
int fsx_pointer_device(const void* p, int* device);
/* What a send() source span is: *kind = 0 pageable (or unknown) host memory,
 * 1 pinned host memory (page-locked / registered: the DMA reads it
 * asynchronously), 2 device or managed memory.  Never fails. */
#define FSX_PTR_PAGEABLE 0
#define FSX_PTR_PINNED 1
#define FSX_PTR_DEVICE 2
int fsx_pointer_kind(const void* p, int* kind);
/* Synchronous device->host copy (owning a device payload that must outlive a
 * borrowed span, e.g. backlogged sends, sidecar.hpp:327). */
int fsx_copy_to_host(void* h_dst, const void* d_src, int64_t n);

/* The copy-engine comparator (BASELINE.json configs[4]: "vs cudaMemcpyPeer"):
 * cudaMemcpyAsync(d_dst, d_src, n, cudaMemcpyDefault) on `stream` of src_gpu's
 * device -- a peer copy over NVLink when d_dst is a peer or IPC-mapped slab.
 * No chunk flags, no digest: timed beside K1 for the same bytes. */
int fsx_copy_engine(fsx_fabric* f, int src_gpu, void* d_dst, const void* d_src, int64_t n,
                    void* stream);

/* ---- stats ----------------------------------------------------------------
 * SidecarStats (sidecar.hpp:209-217, 403-415) device-side counterparts plus
 * the number of fsx kernels launched (bench "gpu_launches"). */
typedef struct fsx_stats {
  int64_t forwards;        /* fsx_forward / fsx_forward_host calls */
  int64_t bytes_forwarded; /* payload bytes moved into slabs */
  int64_t merges;
  int64_t merged_rows;
  int64_t segments_in_use; /* over all slabs */
  int64_t bytes_in_use;
  int64_t kernel_launches;
  int64_t dma_forwards; /* transfers moved by the copy-engine form (FSX_FWD_DMA) */
} fsx_stats;
int fsx_get_stats(fsx_fabric* f, fsx_stats* out);

/* Synchronize every stream the fabric owns. */
int fsx_synchronize(fsx_fabric* f);

#ifdef __cplusplus
}
#endif
#endif /* FSX_H */
