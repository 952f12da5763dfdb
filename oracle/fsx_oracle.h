/*
 * fsx_oracle.h -- CPU restatement of the reference (fissim) sidecar data-plane
 * arithmetic.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * leg may load this library, and only as the checker or the timed CPU baseline.
 * The product (libfsx) never links, loads or calls it.
 *
 * Every function cites the reference file:line it restates; paths are relative
 * to /root/reference/proj.  Parity status:
 *   - or_checksum64 / or_synth_payload_into / or_fnv1a64 / or_splitmix64 /
 *     or_payload_seed / or_item_tokens: PINNED -- checked against vectors
 *     produced by the reference's own functions (oracle/_ref, built unmodified
 *     from the include/fissim headers) committed in tests/golden/.
 *   - or_arena_*: PINNED against the reference NodeArena through oracle/_ref.
 *   - or_merge_*: the reference has NO merge (executor_sim.hpp:386 drops the
 *     bytes).  The contract is derived (DESIGN.md "Merge
 *     contract"); its *inputs* are pinned (payload bytes, row counts, slot
 *     order) but the merged layout itself is "parity unpinned" by the reference.
 */
#ifndef FSX_ORACLE_H
#define FSX_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* common.hpp:203-208 */
uint64_t or_splitmix64(uint64_t* state);
/* common.hpp:210-217 */
uint64_t or_fnv1a64(const char* s, size_t n);
/* common.hpp:221-241 */
uint64_t or_checksum64(const uint8_t* data, size_t len);
/* common.hpp:247-259 */
void or_synth_payload_into(uint64_t seed, uint8_t* out, size_t n);
/* fsx dg64 device digest (fsx's own definition, include/fsx.h "integrity
 * digest"; NOT a reference function -- the reference's checksum64 is serial).
 * Plain sequential restatement used to check the fused K1 digest and
 * fsx_digest bit-exactly. */
uint64_t or_digest64(const uint8_t* data, size_t len);
/* executor_sim.hpp:231-233 */
uint64_t or_payload_seed(const char* ref_id, size_t n, int64_t seq);

/* profiles.hpp:256-276 (ShapeRules::item_tokens).  modality: 0 text, 1 image,
 * 2 video, 3 audio.  Negative width/height/frames or NaN seconds select the
 * ShapeRules defaults passed in `rules` (same order as profiles.hpp:213-226). */
typedef struct or_shape_rules {
  int64_t pixels_per_token;
  int64_t default_image_width;
  int64_t default_image_height;
  int64_t tokens_per_frame;
  int64_t default_video_frames;
  int64_t tokens_per_audio_second;
  double default_audio_seconds;
  int64_t hidden_dim;
  int64_t embed_elem_bytes;
} or_shape_rules;
void or_shape_rules_default(or_shape_rules* r);
int64_t or_item_tokens(const or_shape_rules* r, int modality, int64_t width, int64_t height,
                       int64_t frames, double seconds);

/* NodeArena first-fit allocator, sidecar.hpp:106-205 (allocation policy
 * only: 64 B alignment :195, first-fit over offset order :149-163, coalescing
 * free :165-186).  Returns -1 when nothing fits, -2 on double free. */
typedef struct or_arena or_arena;
or_arena* or_arena_new(int64_t capacity);
void or_arena_delete(or_arena* a);
int64_t or_arena_alloc(or_arena* a, int64_t len);
int or_arena_free(or_arena* a, int64_t off);
int64_t or_arena_segments_in_use(const or_arena* a);
int64_t or_arena_bytes_in_use(const or_arena* a);
int64_t or_arena_peak_bytes(const or_arena* a);

/* ---- Merge restatement (derived contract) -----------------
 * Packed batch of R requests.  Request r owns prompt rows
 * [req_row_off[r], req_row_off[r+1]) of `embeds` (row_bytes each) and of
 * `token_ids`, and items [req_item_off[r], req_item_off[r+1]).  Item i has
 * item_rows[i] rows at host pointer item_src[i].  The k-th row of request r
 * whose token id equals placeholder_id receives row k of
 * concat(item_src[first..last]) in item (= input slot) order
 * (record_replay.hpp:404-416).  Text rows are untouched.  A request whose
 * placeholder count differs from the sum of its item rows is left untouched
 * and gets status[r] = 1 (ErrorCode::Validation ordinal 0, +1).
 * Returns the number of invalid requests.  nthreads > 1 splits requests over
 * pthreads (CPU merge on all host cores). */
int or_merge(int32_t num_requests, int64_t row_bytes, int32_t placeholder_id, uint8_t* embeds,
             const int32_t* token_ids, const int64_t* req_row_off, const int64_t* req_item_off,
             const uint8_t* const* item_src, const int64_t* item_rows, int32_t* status,
             int nthreads);

/* Placeholder layout for synthetic prompts (new contract):
 * input_tokens text rows are split into m+1 segments as evenly as possible
 * (earlier segments take the remainder) around m placeholder runs of
 * item_rows[i].  Text ids are the t-th splitmix64 word of the stream seeded
 * with fnv1a64(request_id + "/tok") reduced mod text_vocab (< placeholder_id),
 * so they never equal the placeholder.  Writes T = input_tokens + sum rows ids. */
void or_prompt_tokens(const char* request_id, size_t rid_len, int64_t input_tokens, int32_t m,
                      const int64_t* item_rows, int32_t placeholder_id, int32_t text_vocab,
                      int32_t* out);

#ifdef __cplusplus
}
#endif
#endif
