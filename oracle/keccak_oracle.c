/*
 * oracle/keccak_oracle.c -- CPU restatement of the reference batch-hash path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing under paper_1902_05320_b200/ may link,
 * import or execute this file; only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py use it, and only as the
 * checker (or as the timed CPU baseline), never as the product.
 *
 * Parity status: PINNED.  tests/test_oracle.py checks this file against
 *   - the 892 .rsp vectors of the reference (converted into tests/golden/ by
 *     tests/golden/make_golden.py),
 *   - the FIPS 202 inline KATs of the reference tests (tests/golden/inline_kats.json),
 *   - the Keccak-f[1600](0) 200-byte state,
 *   - the compiled reference itself (oracle/_ref, built from /root/reference
 *     by oracle/Makefile) on randomized batches, when that library is present.
 *
 * Every function cites the reference lines it restates; paths are relative to
 * /root/reference/proj/core.  Plain C11, 64-bit lanes, no SIMD: this is the
 * same arithmetic the reference performs, written independently.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define KO_EXPORT __attribute__((visibility("default")))

/* rho offsets, lane index x + 5y  (src/keccak.cpp:26-32) */
static const unsigned ko_rho[25] = {
    0,  1,  62, 28, 27, 36, 44, 6,  55, 20, 3,  10, 43,
    25, 39, 41, 45, 15, 21, 8,  18, 2,  61, 56, 14};

/* iota round constants  (src/keccak.cpp:34-43) */
static const uint64_t ko_rc[24] = {
    0x0000000000000001ull, 0x0000000000008082ull, 0x800000000000808aull,
    0x8000000080008000ull, 0x000000000000808bull, 0x0000000080000001ull,
    0x8000000080008081ull, 0x8000000000008009ull, 0x000000000000008aull,
    0x0000000000000088ull, 0x0000000080008009ull, 0x000000008000000aull,
    0x000000008000808bull, 0x800000000000008bull, 0x8000000000008089ull,
    0x8000000000008003ull, 0x8000000000008002ull, 0x8000000000000080ull,
    0x000000000000800aull, 0x800000008000000aull, 0x8000000080008081ull,
    0x8000000000008080ull, 0x0000000080000001ull, 0x8000000080008008ull};

/* (capacity bits, suffix|first pad bit, digest bits) per Algorithm enum value
 * 0..5 = sha3_224, sha3_256, sha3_384, sha3_512, shake128, shake256
 * (include/sha3/sha3.hpp:15-22, src/sha3.cpp:13-20).  The pad head byte is
 * suffix | 1<<suffix_bits = 0x06 / 0x1f (src/sponge.cpp:122). */
typedef struct {
  unsigned capacity_bits;
  uint8_t suffix;
  unsigned suffix_bits;
  unsigned digest_bits; /* 0 = XOF */
} ko_variant;

static const ko_variant ko_variants[6] = {
    {448, 0x02, 2, 224}, {512, 0x02, 2, 256},  {768, 0x02, 2, 384},
    {1024, 0x02, 2, 512}, {256, 0x0f, 4, 0},   {512, 0x0f, 4, 0}};

static inline uint64_t ko_rotl(uint64_t v, unsigned n) {
  n &= 63u;
  return n ? (v << n) | (v >> (64u - n)) : v;
}

/* Keccak-f[1600], 24 rounds of theta, rho+pi, chi, iota on 25 lanes indexed
 * x + 5y  (src/keccak.cpp:245-277). */
KO_EXPORT void ko_permute_1600(uint64_t a[25]) {
  for (int round = 0; round < 24; ++round) {
    uint64_t parity[5], plane[25];
    for (int x = 0; x < 5; ++x)
      parity[x] = a[x] ^ a[x + 5] ^ a[x + 10] ^ a[x + 15] ^ a[x + 20];
    for (int x = 0; x < 5; ++x) {
      uint64_t d = parity[(x + 4) % 5] ^ ko_rotl(parity[(x + 1) % 5], 1);
      for (int y = 0; y < 5; ++y) a[x + 5 * y] ^= d;
    }
    for (int x = 0; x < 5; ++x)
      for (int y = 0; y < 5; ++y) {
        int src = (x + 3 * y) % 5 + 5 * x;
        plane[x + 5 * y] = ko_rotl(a[src], ko_rho[src]);
      }
    for (int y = 0; y < 5; ++y)
      for (int x = 0; x < 5; ++x)
        a[x + 5 * y] = plane[x + 5 * y] ^
                       (~plane[(x + 1) % 5 + 5 * y] & plane[(x + 2) % 5 + 5 * y]);
    a[0] ^= ko_rc[round];
  }
}

/* Byte-oriented sponge  (include/sha3/sponge.hpp:38-64). */
typedef struct {
  uint64_t lanes[25];
  unsigned rate_bytes;
  unsigned pos;
  int squeezing;
} ko_sponge;

/* src/sponge.cpp:71-75, :145-149 */
static void ko_sponge_init(ko_sponge* s, unsigned rate_bytes) {
  memset(s->lanes, 0, sizeof s->lanes);
  s->rate_bytes = rate_bytes;
  s->pos = 0;
  s->squeezing = 0;
}

/* src/sponge.cpp:81-111: XOR bytes little-endian into the rate part, permute
 * every time the block fills.  (The reference has an 8-byte memcpy fast path;
 * the byte loop below is arithmetically identical.) */
static void ko_sponge_update(ko_sponge* s, const uint8_t* p, uint64_t n) {
  while (n > 0) {
    if ((s->pos & 7u) == 0 && n >= 8 && s->pos + 8 <= (s->rate_bytes & ~7u)) {
      uint64_t v;
      memcpy(&v, p, 8); /* host is little-endian, like the reference assumes */
      s->lanes[s->pos >> 3] ^= v;
      s->pos += 8;
      p += 8;
      n -= 8;
    } else {
      s->lanes[s->pos >> 3] ^= (uint64_t)(*p) << ((s->pos & 7u) * 8u);
      s->pos += 1;
      p += 1;
      n -= 1;
    }
    if (s->pos == s->rate_bytes) {
      ko_permute_1600(s->lanes);
      s->pos = 0;
    }
  }
}

/* src/sponge.cpp:113-129 */
static void ko_sponge_finish(ko_sponge* s, uint8_t domain, unsigned domain_bits) {
  uint8_t head = (uint8_t)(domain | (1u << domain_bits));
  unsigned last = s->rate_bytes - 1;
  s->lanes[s->pos >> 3] ^= (uint64_t)head << ((s->pos & 7u) * 8u);
  s->lanes[last >> 3] ^= 0x80ull << ((last & 7u) * 8u);
  ko_permute_1600(s->lanes);
  s->pos = 0;
  s->squeezing = 1;
}

/* src/sponge.cpp:131-143 */
static void ko_sponge_squeeze(ko_sponge* s, uint8_t* out, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) {
    if (s->pos == s->rate_bytes) {
      ko_permute_1600(s->lanes);
      s->pos = 0;
    }
    out[i] = (uint8_t)(s->lanes[s->pos >> 3] >> ((s->pos & 7u) * 8u));
    s->pos += 1;
  }
}

/* rate in bytes = (1600 - capacity)/8  (include/sha3/sha3.hpp:40) */
KO_EXPORT unsigned ko_rate_bytes(int algorithm) {
  if (algorithm < 0 || algorithm > 5) return 0;
  return (1600u - ko_variants[algorithm].capacity_bits) / 8u;
}

/* src/batch.cpp:74-75 */
KO_EXPORT uint64_t ko_digest_bytes(int algorithm, uint64_t xof_bits) {
  if (algorithm < 0 || algorithm > 5) return 0;
  const ko_variant* v = &ko_variants[algorithm];
  return v->digest_bits == 0 ? (xof_bits + 7) / 8 : v->digest_bits / 8;
}

/* One message: src/batch.cpp:15-25 (identical sequence to sha3_digest / shake,
 * src/sha3.cpp:60-93). */
KO_EXPORT int ko_hash_one(int algorithm, uint64_t xof_bits, const uint8_t* msg,
                          uint64_t len, uint8_t* out) {
  if (algorithm < 0 || algorithm > 5) return 1;
  const ko_variant* v = &ko_variants[algorithm];
  if (v->digest_bits == 0 && xof_bits == 0) return 1;
  uint64_t nout = ko_digest_bytes(algorithm, xof_bits);
  ko_sponge s;
  ko_sponge_init(&s, ko_rate_bytes(algorithm));
  ko_sponge_update(&s, msg, len);
  ko_sponge_finish(&s, v->suffix, v->suffix_bits);
  ko_sponge_squeeze(&s, out, nout);
  if (v->digest_bits == 0 && (xof_bits % 8) != 0)
    out[nout - 1] &= (uint8_t)((1u << (xof_bits % 8)) - 1u);
  return 0;
}

/* Batch over a packed buffer.  Semantics of src/batch.cpp:64-135: validation
 * before any work, digest i belongs to message i, contiguous chunks handed to
 * workers through a shared cursor (:94-127; auto chunk = ceil(n / (8*workers)),
 * :46-62).  offsets == NULL means fixed-length messages at i*lengths[0]. */
typedef struct {
  int algorithm;
  uint64_t xof_bits;
  const uint8_t* data;
  const uint64_t* offsets;
  const uint64_t* lengths;
  uint64_t fixed_len;
  uint64_t count;
  uint64_t chunk;
  uint64_t digest_bytes;
  uint8_t* out;
  uint64_t cursor; /* accessed with __atomic builtins */
} ko_job;

static void* ko_worker(void* arg) {
  ko_job* job = (ko_job*)arg;
  for (;;) {
    uint64_t begin = __atomic_fetch_add(&job->cursor, job->chunk, __ATOMIC_RELAXED);
    if (begin >= job->count) return NULL;
    uint64_t end = begin + job->chunk < job->count ? begin + job->chunk : job->count;
    for (uint64_t i = begin; i < end; ++i) {
      uint64_t off = job->offsets ? job->offsets[i] : i * job->fixed_len;
      uint64_t len = job->lengths ? job->lengths[i] : job->fixed_len;
      ko_hash_one(job->algorithm, job->xof_bits, job->data + off, len,
                  job->out + i * job->digest_bytes);
    }
  }
}

KO_EXPORT int ko_hash_batch(int algorithm, const uint8_t* data,
                            const uint64_t* offsets, const uint64_t* lengths,
                            uint64_t fixed_len, uint64_t count, uint64_t xof_bits,
                            uint8_t* out, unsigned workers) {
  if (algorithm < 0 || algorithm > 5) return 1;
  if (ko_variants[algorithm].digest_bits == 0 && xof_bits == 0) return 1;
  if (count == 0) return 0;
  if (workers == 0) workers = 1;
  ko_job job;
  job.algorithm = algorithm;
  job.xof_bits = xof_bits;
  job.data = data;
  job.offsets = offsets;
  job.lengths = lengths;
  job.fixed_len = fixed_len;
  job.count = count;
  job.chunk = (count + 8ull * workers - 1) / (8ull * workers);
  if (job.chunk == 0) job.chunk = 1;
  job.digest_bytes = ko_digest_bytes(algorithm, xof_bits);
  job.out = out;
  job.cursor = 0;
  if (workers == 1) {
    ko_worker(&job);
    return 0;
  }
  pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * (workers - 1));
  unsigned started = 0;
  for (unsigned t = 0; t + 1 < workers; ++t)
    if (pthread_create(&tids[started], NULL, ko_worker, &job) == 0) ++started;
  ko_worker(&job); /* the caller participates (src/batch.cpp:126) */
  for (unsigned t = 0; t < started; ++t) pthread_join(tids[t], NULL);
  free(tids);
  return 0;
}

/* splitmix64 (tools/sha3cli/workload.hpp:25-36, tests/test_util.hpp:14-27) */
static inline uint64_t ko_splitmix_next(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

/* Fixed-size synthetic messages, packed back to back
 * (tools/sha3cli/workload.cpp:16-47): generator seeded with
 * seed ^ total_bytes*gamma; ceil(size/8) words per message, little-endian,
 * surplus bytes of the last word dropped.  Returns the message count. */
KO_EXPORT uint64_t ko_generate_workload(uint64_t seed, uint64_t total_bytes,
                                        uint64_t message_size, uint8_t* out) {
  if (message_size == 0 || total_bytes < message_size) return 0;
  uint64_t count = total_bytes / message_size;
  uint64_t state = seed ^ (total_bytes * 0x9e3779b97f4a7c15ull);
  for (uint64_t m = 0; m < count; ++m) {
    uint8_t* msg = out + m * message_size;
    uint64_t i = 0;
    while (i < message_size) {
      uint64_t word = ko_splitmix_next(&state);
      for (int k = 0; k < 8 && i < message_size; ++k, ++i)
        msg[i] = (uint8_t)(word >> (8 * k));
    }
  }
  return count;
}

/* Test-data generator of the reference tests: one splitmix64 draw per byte
 * (tests/test_util.hpp:29-35) and below(n) = next() % n (:26).  The state is
 * passed in and out so that Python can interleave the two like the tests do. */
KO_EXPORT uint64_t ko_testrng_below(uint64_t* state, uint64_t n) {
  return ko_splitmix_next(state) % n;
}

KO_EXPORT void ko_testrng_bytes(uint64_t* state, uint8_t* out, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) out[i] = (uint8_t)ko_splitmix_next(state);
}
