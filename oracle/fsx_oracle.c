/*
 * fsx_oracle.c -- CPU restatement of the reference sidecar data-plane
 * arithmetic.  TEST INFRASTRUCTURE ONLY (see fsx_oracle.h for the rules and
 * the parity status of each function).  Plain C11, no dependencies.
 */
#include "fsx_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------------
 * Hashing / synthesis primitives */

/* common.hpp:203-208: state advances by the golden gamma, then two
 * xor-shift-multiply rounds and a final xor-shift. */
uint64_t or_splitmix64(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

/* common.hpp:210-217: FNV-1a, 64-bit offset basis and prime. */
uint64_t or_fnv1a64(const char* s, size_t n) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (size_t i = 0; i < n; ++i) {
    h ^= (unsigned char)s[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

static uint64_t load_le64(const uint8_t* p) {
  uint64_t v = 0;
  for (int b = 7; b >= 0; --b) v = (v << 8) | p[b];
  return v;
}

/* common.hpp:221-241: seeded with the length, one multiply/xorshift round per
 * little-endian 8-byte lane (:224-230), tail bytes packed little-endian
 * (:231-237), final round with a 32-bit shift (:238-239). */
uint64_t or_checksum64(const uint8_t* data, size_t len) {
  const uint64_t k = 0x2545f4914f6cdd1dull;
  uint64_t h = 0x9e3779b97f4a7c15ull ^ ((uint64_t)len * 0xff51afd7ed558ccdull);
  size_t i = 0;
  for (; i + 8 <= len; i += 8) {
    h = (h ^ load_le64(data + i)) * k;
    h ^= h >> 29;
  }
  uint64_t tail = 0;
  for (int shift = 0; i < len; ++i, shift += 8) tail |= (uint64_t)data[i] << shift;
  h = (h ^ tail) * k;
  h ^= h >> 32;
  return h;
}

/* common.hpp:247-259: splitmix64 stream from seed ^ 0xd6e8feb86659fd93,
 * words stored little-endian, the tail is a truncated next word. */
void or_synth_payload_into(uint64_t seed, uint8_t* out, size_t n) {
  uint64_t s = seed ^ 0xd6e8feb86659fd93ull;
  size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    uint64_t v = or_splitmix64(&s);
    for (int b = 0; b < 8; ++b) out[i + b] = (uint8_t)(v >> (8 * b));
  }
  if (i < n) {
    uint64_t v = or_splitmix64(&s);
    for (int b = 0; i < n; ++i, ++b) out[i] = (uint8_t)(v >> (8 * b));
  }
}

/* fsx dg64 (include/fsx.h): n*G + sum over LE words of f(w ^ (k+1)*C1). */
uint64_t or_digest64(const uint8_t* data, size_t len) {
  uint64_t h = (uint64_t)len * 0x9e3779b97f4a7c15ull;
  for (size_t k = 0; k * 8 < len; ++k) {
    uint64_t w = 0;
    for (size_t b = 0; b < 8 && k * 8 + b < len; ++b) w |= (uint64_t)data[k * 8 + b] << (8 * b);
    uint64_t y = (w ^ ((uint64_t)(k + 1) * 0xbf58476d1ce4e5b9ull)) * 0x94d049bb133111ebull;
    h += y ^ (y >> 29);
  }
  return h;
}

/* executor_sim.hpp:231-233 */
uint64_t or_payload_seed(const char* ref_id, size_t n, int64_t seq) {
  return or_fnv1a64(ref_id, n) ^ (0x9e3779b97f4a7c15ull * (uint64_t)(seq + 1));
}

/* ---------------------------------------------------------------------------
 * Shape rules */

/* profiles.hpp:213-226 field defaults */
void or_shape_rules_default(or_shape_rules* r) {
  r->pixels_per_token = 1024;
  r->default_image_width = 896;
  r->default_image_height = 896;
  r->tokens_per_frame = 196;
  r->default_video_frames = 16;
  r->tokens_per_audio_second = 25;
  r->default_audio_seconds = 8;
  r->hidden_dim = 1024;
  r->embed_elem_bytes = 2;
}

/* profiles.hpp:256-276 */
int64_t or_item_tokens(const or_shape_rules* r, int modality, int64_t width, int64_t height,
                       int64_t frames, double seconds) {
  switch (modality) {
    case 1: {
      int64_t w = width < 0 ? r->default_image_width : width;
      int64_t h = height < 0 ? r->default_image_height : height;
      return (w * h + r->pixels_per_token - 1) / r->pixels_per_token;
    }
    case 2:
      return (frames < 0 ? r->default_video_frames : frames) * r->tokens_per_frame;
    case 3: {
      double s = isnan(seconds) ? r->default_audio_seconds : seconds;
      return (int64_t)ceil(s * (double)r->tokens_per_audio_second);
    }
    default:
      return 0;
  }
}

/* ---------------------------------------------------------------------------
 * First-fit arena (allocation policy of sidecar.hpp:106-205).  Sorted arrays
 * of (offset, length) for the free and used lists. */

typedef struct {
  int64_t off, len;
} seg_t;

typedef struct {
  seg_t* v;
  size_t n, cap;
} seglist;

struct or_arena {
  int64_t capacity, in_use, peak;
  seglist free_, used_;
};

static size_t seg_lower(const seglist* l, int64_t off) {
  size_t lo = 0, hi = l->n;
  while (lo < hi) {
    size_t mid = (lo + hi) / 2;
    if (l->v[mid].off < off) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

static void seg_insert(seglist* l, int64_t off, int64_t len) {
  if (l->n == l->cap) {
    l->cap = l->cap ? l->cap * 2 : 16;
    l->v = (seg_t*)realloc(l->v, l->cap * sizeof(seg_t));
  }
  size_t at = seg_lower(l, off);
  memmove(l->v + at + 1, l->v + at, (l->n - at) * sizeof(seg_t));
  l->v[at].off = off;
  l->v[at].len = len;
  l->n++;
}

static void seg_erase(seglist* l, size_t at) {
  memmove(l->v + at, l->v + at + 1, (l->n - at - 1) * sizeof(seg_t));
  l->n--;
}

or_arena* or_arena_new(int64_t capacity) {
  or_arena* a = (or_arena*)calloc(1, sizeof(or_arena));
  a->capacity = capacity;
  seg_insert(&a->free_, 0, capacity);
  return a;
}

void or_arena_delete(or_arena* a) {
  if (!a) return;
  free(a->free_.v);
  free(a->used_.v);
  free(a);
}

/* sidecar.hpp:149-163 (zero-byte requests take one aligned unit, :150) */
int64_t or_arena_alloc(or_arena* a, int64_t len) {
  int64_t need = ((len < 1 ? 1 : len) + 63) & ~(int64_t)63;
  for (size_t i = 0; i < a->free_.n; ++i) {
    if (a->free_.v[i].len < need) continue;
    int64_t off = a->free_.v[i].off, rest = a->free_.v[i].len - need;
    seg_erase(&a->free_, i);
    if (rest > 0) seg_insert(&a->free_, off + need, rest);
    seg_insert(&a->used_, off, need);
    a->in_use += need;
    if (a->in_use > a->peak) a->peak = a->in_use;
    return off;
  }
  return -1;
}

/* sidecar.hpp:165-186 */
int or_arena_free(or_arena* a, int64_t off) {
  size_t u = seg_lower(&a->used_, off);
  if (u >= a->used_.n || a->used_.v[u].off != off) return -2;
  int64_t len = a->used_.v[u].len;
  seg_erase(&a->used_, u);
  a->in_use -= len;
  size_t nx = seg_lower(&a->free_, off);
  if (nx < a->free_.n && a->free_.v[nx].off == off + len) {
    len += a->free_.v[nx].len;
    seg_erase(&a->free_, nx);
  }
  if (nx > 0 && a->free_.v[nx - 1].off + a->free_.v[nx - 1].len == off) {
    off = a->free_.v[nx - 1].off;
    len += a->free_.v[nx - 1].len;
    seg_erase(&a->free_, nx - 1);
  }
  seg_insert(&a->free_, off, len);
  return 0;
}

int64_t or_arena_segments_in_use(const or_arena* a) { return (int64_t)a->used_.n; }
int64_t or_arena_bytes_in_use(const or_arena* a) { return a->in_use; }
int64_t or_arena_peak_bytes(const or_arena* a) { return a->peak; }

/* ---------------------------------------------------------------------------
 * Merge restatement (derived contract; see header). */

typedef struct {
  int32_t r0, r1;
  int64_t row_bytes;
  int32_t pid;
  uint8_t* embeds;
  const int32_t* tok;
  const int64_t* req_row_off;
  const int64_t* req_item_off;
  const uint8_t* const* item_src;
  const int64_t* item_rows;
  int32_t* status;
  int bad;
} merge_job;

static void merge_one(const merge_job* j, int32_t r, int* bad) {
  int64_t t0 = j->req_row_off[r], t1 = j->req_row_off[r + 1];
  int64_t i0 = j->req_item_off[r], i1 = j->req_item_off[r + 1];
  int64_t want = 0, have = 0;
  for (int64_t i = i0; i < i1; ++i) want += j->item_rows[i];
  for (int64_t t = t0; t < t1; ++t) have += j->tok[t] == j->pid;
  if (want != have) {
    j->status[r] = 1; /* 1 + ErrorCode::Validation (common.hpp:29-30) */
    ++*bad;
    return;
  }
  j->status[r] = 0;
  int64_t item = i0, row_in_item = 0;
  for (int64_t t = t0; t < t1; ++t) {
    if (j->tok[t] != j->pid) continue;
    while (row_in_item == j->item_rows[item]) {
      ++item;
      row_in_item = 0;
    }
    memcpy(j->embeds + t * j->row_bytes, j->item_src[item] + row_in_item * j->row_bytes,
           (size_t)j->row_bytes);
    ++row_in_item;
  }
}

static void* merge_worker(void* p) {
  merge_job* j = (merge_job*)p;
  for (int32_t r = j->r0; r < j->r1; ++r) merge_one(j, r, &j->bad);
  return NULL;
}

int or_merge(int32_t num_requests, int64_t row_bytes, int32_t placeholder_id, uint8_t* embeds,
             const int32_t* token_ids, const int64_t* req_row_off, const int64_t* req_item_off,
             const uint8_t* const* item_src, const int64_t* item_rows, int32_t* status,
             int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > num_requests) nthreads = num_requests > 0 ? num_requests : 1;
  merge_job proto = {0, 0, row_bytes, placeholder_id, embeds, token_ids, req_row_off,
                     req_item_off, item_src, item_rows, status, 0};
  if (nthreads == 1) {
    proto.r1 = num_requests;
    merge_worker(&proto);
    return proto.bad;
  }
  merge_job* jobs = (merge_job*)calloc((size_t)nthreads, sizeof(merge_job));
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  int32_t per = num_requests / nthreads, extra = num_requests % nthreads, at = 0;
  for (int k = 0; k < nthreads; ++k) {
    jobs[k] = proto;
    jobs[k].r0 = at;
    at += per + (k < extra ? 1 : 0);
    jobs[k].r1 = at;
    pthread_create(&th[k], NULL, merge_worker, &jobs[k]);
  }
  int bad = 0;
  for (int k = 0; k < nthreads; ++k) {
    pthread_join(th[k], NULL);
    bad += jobs[k].bad;
  }
  free(jobs);
  free(th);
  return bad;
}

/* ---------------------------------------------------------------------------
 * Synthetic prompt token layout (new contract). */
void or_prompt_tokens(const char* request_id, size_t rid_len, int64_t input_tokens, int32_t m,
                      const int64_t* item_rows, int32_t placeholder_id, int32_t text_vocab,
                      int32_t* out) {
  char buf[512];
  size_t n = rid_len < sizeof(buf) - 8 ? rid_len : sizeof(buf) - 8;
  memcpy(buf, request_id, n);
  memcpy(buf + n, "/tok", 4);
  uint64_t s = or_fnv1a64(buf, n + 4) ^ 0xd6e8feb86659fd93ull;
  int64_t segs = (int64_t)m + 1, base = input_tokens / segs, rem = input_tokens % segs;
  int64_t t = 0;
  for (int64_t seg = 0; seg < segs; ++seg) {
    int64_t len = base + (seg < rem ? 1 : 0);
    for (int64_t k = 0; k < len; ++k, ++t)
      out[t] = (int32_t)(or_splitmix64(&s) % (uint64_t)text_vocab);
    if (seg < m) {
      for (int64_t k = 0; k < item_rows[seg]; ++k, ++t) {
        (void)or_splitmix64(&s); /* one word per row keeps ids position-determined */
        out[t] = placeholder_id;
      }
    }
  }
}
