/*
 * gompgen.c — seeded synthetic input generators shared by the oracle tests and the CUDA-path tests/bench.
 *
 * This module holds NONE of the method's arithmetic (no LZ77, no Huffman, no format code): it only
 * produces uncompressed byte strings with the shape of the paper's workloads (DESIGN.md §4 recipe):
 *
 *   gg_wiki    Wikipedia-XML-shaped text  (paper dataset 1: "1 GB XML dump of the English Wikipedia",
 *              PAPER.md:541-545; calibrated to gzip -6 ≈ 3.1)
 *   gg_text    English-like article text only (config C1)
 *   gg_matrix  MatrixMarket coordinate text (paper dataset 2: "Hollywood-2009" CSV)
 *   gg_nested  the nesting-depth dataset of P:583-613 (Fig. 32nesting): a 16-byte string repeated with a
 *              one-byte change alternating between the first and last byte, a separator byte from a
 *              disjoint set after every instance, 32/D distinct strings interleaved for depth D
 *   gg_random  uniformly random bytes (incompressible edge case)
 *
 * Every generator is a pure function of (seed, n, params): xoshiro256** seeded through splitmix64.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { uint64_t s[4]; } rng_t;

static uint64_t splitmix64(uint64_t *x) {
  uint64_t z = (*x += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static void rng_seed(rng_t *r, uint64_t seed) {
  uint64_t x = seed;
  for (int i = 0; i < 4; i++) r->s[i] = splitmix64(&x);
}
static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static uint64_t rng_next(rng_t *r) {
  uint64_t *s = r->s;
  uint64_t res = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
  s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t; s[3] = rotl(s[3], 45);
  return res;
}
static double rng_unif(rng_t *r) { return (double)(rng_next(r) >> 11) * (1.0 / 9007199254740992.0); }
static uint32_t rng_below(rng_t *r, uint32_t n) { return (uint32_t)(((rng_next(r) >> 32) * (uint64_t)n) >> 32); }
static double rng_normal(rng_t *r) {
  double u1 = rng_unif(r), u2 = rng_unif(r);
  if (u1 < 1e-300) u1 = 1e-300;
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

/* ---------------------------------------------------------------- output buffer */
typedef struct { uint8_t *p; uint64_t n, cap; } obuf_t;
static inline int ob_full(const obuf_t *o) { return o->n >= o->cap; }
static void ob_put(obuf_t *o, const char *s, size_t len) {
  size_t k = len;
  if (o->n + k > o->cap) k = (size_t)(o->cap - o->n);
  memcpy(o->p + o->n, s, k);
  o->n += k;
}
static void ob_str(obuf_t *o, const char *s) { ob_put(o, s, strlen(s)); }
static void ob_uint(obuf_t *o, uint64_t v) {
  char tmp[24];
  int k = 0;
  do { tmp[k++] = (char)('0' + v % 10); v /= 10; } while (v);
  char out[24];
  for (int i = 0; i < k; i++) out[i] = tmp[k - 1 - i];
  ob_put(o, out, (size_t)k);
}

/* ---------------------------------------------------------------- vocabulary (wiki/text) */
#define NWORDS 60000
typedef struct {
  char *pool;        /* all words, NUL-separated */
  uint32_t off[NWORDS];
  uint8_t len[NWORDS];
  double *cdf;       /* Zipf(s=1.2) cumulative distribution over word ranks */
} vocab_t;

static void vocab_build(vocab_t *v, rng_t *r) {
  static const char cons[] = "bcdfghjklmnprstvwz";
  static const char vows[] = "aeiou";
  v->pool = (char *)malloc((size_t)NWORDS * 17);
  uint32_t at = 0;
  for (int w = 0; w < NWORDS; w++) {
    double l = exp(1.6 + 0.45 * rng_normal(r));
    int len = (int)(l + 0.5);
    if (len < 1) len = 1;
    if (len > 15) len = 15;
    int start_vowel = (int)rng_below(r, 3) == 0;
    v->off[w] = at;
    v->len[w] = (uint8_t)len;
    for (int i = 0; i < len; i++) {
      int vowel = ((i & 1) == 0) == start_vowel;
      v->pool[at++] = vowel ? vows[rng_below(r, 5)] : cons[rng_below(r, 18)];
    }
    v->pool[at++] = 0;
  }
  v->cdf = (double *)malloc(sizeof(double) * NWORDS);
  double acc = 0;
  for (int w = 0; w < NWORDS; w++) { acc += 1.0 / pow((double)(w + 1), 1.2); v->cdf[w] = acc; }
  for (int w = 0; w < NWORDS; w++) v->cdf[w] /= acc;
}
static void vocab_free(vocab_t *v) { free(v->pool); free(v->cdf); }
static int vocab_pick(const vocab_t *v, rng_t *r) {
  double u = rng_unif(r);
  int lo = 0, hi = NWORDS - 1;
  while (lo < hi) { int mid = (lo + hi) >> 1; if (v->cdf[mid] < u) lo = mid + 1; else hi = mid; }
  return lo;
}
static void ob_word(obuf_t *o, const vocab_t *v, int w, int cap) {
  const char *s = v->pool + v->off[w];
  if (cap && s[0] >= 'a' && s[0] <= 'z') {
    char c = (char)(s[0] - 32);
    ob_put(o, &c, 1);
    ob_put(o, s + 1, v->len[w] - 1u);
  } else {
    ob_put(o, s, v->len[w]);
  }
}

/* one sentence of article text with wiki markup */
static void gen_sentence(obuf_t *o, const vocab_t *v, rng_t *r, int markup) {
  int nw = 4 + (int)rng_below(r, 18);
  for (int i = 0; i < nw && !ob_full(o); i++) {
    if (i) ob_str(o, " ");
    double u = rng_unif(r);
    int w = vocab_pick(v, r);
    if (markup && u < 0.06) { ob_str(o, "[["); ob_word(o, v, w, 1); ob_str(o, "]]"); }
    else if (markup && u < 0.08) {
      ob_str(o, "[["); ob_word(o, v, w, 1); ob_str(o, " "); ob_word(o, v, vocab_pick(v, r), 0);
      ob_str(o, "|"); ob_word(o, v, w, 0); ob_str(o, "]]");
    } else if (markup && u < 0.09) { ob_str(o, "'''"); ob_word(o, v, w, i == 0); ob_str(o, "'''"); }
    else if (u < 0.10) { ob_uint(o, rng_below(r, 3000)); }
    else ob_word(o, v, w, i == 0);
    if (i + 1 < nw && rng_below(r, 12) == 0) ob_str(o, ",");
  }
  ob_str(o, ".");
  if (markup && rng_below(r, 20) == 0) {
    ob_str(o, "&lt;ref&gt;{{cite web |url=http://www.");
    ob_word(o, v, vocab_pick(v, r), 0); ob_str(o, ".com/"); ob_word(o, v, vocab_pick(v, r), 0);
    ob_str(o, ".html |title="); ob_word(o, v, vocab_pick(v, r), 1); ob_str(o, " ");
    ob_word(o, v, vocab_pick(v, r), 0); ob_str(o, " |accessdate=");
    ob_uint(o, 2000 + rng_below(r, 16)); ob_str(o, "-");
    uint32_t m = 1 + rng_below(r, 12), d = 1 + rng_below(r, 28);
    if (m < 10) ob_str(o, "0");
    ob_uint(o, m); ob_str(o, "-");
    if (d < 10) ob_str(o, "0");
    ob_uint(o, d); ob_str(o, "}}&lt;/ref&gt;");
  }
}

static void gen_article(obuf_t *o, const vocab_t *v, rng_t *r, int markup) {
  int np = 2 + (int)rng_below(r, 11);
  for (int p = 0; p < np && !ob_full(o); p++) {
    if (markup && p > 0 && rng_unif(r) < 0.30) {
      int lvl = 2 + (int)rng_below(r, 2);
      for (int i = 0; i < lvl; i++) ob_str(o, "=");
      ob_str(o, " "); ob_word(o, v, vocab_pick(v, r), 1); ob_str(o, " ");
      ob_word(o, v, vocab_pick(v, r), 0); ob_str(o, " ");
      for (int i = 0; i < lvl; i++) ob_str(o, "=");
      ob_str(o, "\n");
    }
    int ns = 1 + (int)rng_below(r, 7);
    for (int s = 0; s < ns && !ob_full(o); s++) {
      if (s) ob_str(o, " ");
      gen_sentence(o, v, r, markup);
    }
    ob_str(o, "\n\n");
  }
}

/* Wikipedia-shaped XML dump (paper dataset 1) */
int gg_wiki(uint64_t seed, uint8_t *dst, uint64_t n) {
  rng_t r; rng_seed(&r, seed);
  vocab_t v; vocab_build(&v, &r);
  obuf_t o = {dst, 0, n};
  uint64_t id = 10 + rng_below(&r, 1000), rev = 100000 + rng_below(&r, 100000);
  ob_str(&o, "<mediawiki xml:lang=\"en\">\n");
  while (!ob_full(&o)) {
    ob_str(&o, "  <page>\n    <title>");
    ob_word(&o, &v, vocab_pick(&v, &r), 1); ob_str(&o, " ");
    ob_word(&o, &v, vocab_pick(&v, &r), 1);
    ob_str(&o, "</title>\n    <ns>0</ns>\n    <id>"); ob_uint(&o, id);
    ob_str(&o, "</id>\n    <revision>\n      <id>"); ob_uint(&o, rev);
    ob_str(&o, "</id>\n      <timestamp>");
    ob_uint(&o, 2001 + rng_below(&r, 15)); ob_str(&o, "-0"); ob_uint(&o, 1 + rng_below(&r, 9));
    ob_str(&o, "-1"); ob_uint(&o, rng_below(&r, 10)); ob_str(&o, "T0"); ob_uint(&o, rng_below(&r, 10));
    ob_str(&o, ":1"); ob_uint(&o, rng_below(&r, 10)); ob_str(&o, ":2"); ob_uint(&o, rng_below(&r, 10));
    ob_str(&o, "Z</timestamp>\n      <contributor>\n        <username>");
    ob_word(&o, &v, vocab_pick(&v, &r), 1); ob_uint(&o, rng_below(&r, 100));
    ob_str(&o, "</username>\n        <id>"); ob_uint(&o, 1000 + rng_below(&r, 900000));
    ob_str(&o, "</id>\n      </contributor>\n      <text xml:space=\"preserve\">");
    gen_article(&o, &v, &r, 1);
    int nc = (int)rng_below(&r, 5);
    for (int c = 0; c < nc; c++) {
      ob_str(&o, "[[Category:"); ob_word(&o, &v, vocab_pick(&v, &r), 1); ob_str(&o, " ");
      ob_word(&o, &v, vocab_pick(&v, &r), 0); ob_str(&o, "]]\n");
    }
    ob_str(&o, "</text>\n    </revision>\n  </page>\n");
    id += 1 + rng_below(&r, 40);
    rev += 1 + rng_below(&r, 5000);
  }
  vocab_free(&v);
  return 0;
}

/* English-like article text only (config C1) */
int gg_text(uint64_t seed, uint8_t *dst, uint64_t n) {
  rng_t r; rng_seed(&r, seed);
  vocab_t v; vocab_build(&v, &r);
  obuf_t o = {dst, 0, n};
  while (!ob_full(&o)) gen_article(&o, &v, &r, 0);
  vocab_free(&v);
  return 0;
}

/* MatrixMarket coordinate text, Hollywood-2009-shaped (paper dataset 2) */
static int cmp_u32(const void *a, const void *b) {
  uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
  return (x > y) - (x < y);
}
int gg_matrix(uint64_t seed, uint8_t *dst, uint64_t n) {
  rng_t r; rng_seed(&r, seed);
  obuf_t o = {dst, 0, n};
  const uint32_t N = 1139905;
  ob_str(&o, "%%MatrixMarket matrix coordinate pattern symmetric\n");
  ob_uint(&o, N); ob_str(&o, " "); ob_uint(&o, N); ob_str(&o, " 57515616\n");
  uint32_t cols[4096];
  for (uint32_t row = 1; !ob_full(&o); row = row % N + 1) {
    /* Pareto(alpha = 1.8) degree, scale 20 (gzip -6 ≈ 4.9, the paper's Matrix is 4.99), capped */
    double u = rng_unif(&r);
    if (u < 1e-12) u = 1e-12;
    uint32_t deg = (uint32_t)(20.0 * pow(u, -1.0 / 1.8));
    if (deg > 4096) deg = 4096;
    if (deg < 1) deg = 1;
    uint32_t ncent = 1 + rng_below(&r, 4);
    uint32_t cent[4];
    for (uint32_t k = 0; k < ncent; k++) cent[k] = 1 + rng_below(&r, N);
    for (uint32_t i = 0; i < deg; i++) {
      double c = (double)cent[rng_below(&r, ncent)] + 40.0 * rng_normal(&r);
      if (c < 1) c = 1;
      if (c > N) c = N;
      cols[i] = (uint32_t)c;
    }
    qsort(cols, deg, sizeof(uint32_t), cmp_u32);
    for (uint32_t i = 0; i < deg && !ob_full(&o); i++) {
      if (i && cols[i] == cols[i - 1]) continue;
      ob_uint(&o, cols[i]); ob_str(&o, " "); ob_uint(&o, row); ob_str(&o, "\n");
    }
  }
  return 0;
}

/*
 * Nesting-depth dataset. D in {1,2,4,8,16,32}; k = 32/D distinct 16-byte strings, emitted
 * round-robin. Each new instance of string j differs from its previous instance in one byte, alternately
 * the first and the last; every instance is followed by a separator byte from the disjoint set 249..255.
 */
int gg_nested(uint64_t seed, uint8_t *dst, uint64_t n, uint32_t depth) {
  if (depth == 0 || depth > 32 || (32 % depth) != 0) return -1;
  uint32_t k = 32 / depth;
  uint8_t str[32][16];
  uint32_t cf[32], cl[32], flip[32];
  rng_t r; rng_seed(&r, seed);
  uint32_t salt = rng_below(&r, 249);
  for (uint32_t j = 0; j < k; j++) {
    for (uint32_t i = 0; i < 16; i++) str[j][i] = (uint8_t)((17 * j + 31 * i + 1 + salt) % 249);
    cf[j] = 0; cl[j] = 0; flip[j] = 0;
  }
  obuf_t o = {dst, 0, n};
  for (uint64_t u = 0; !ob_full(&o); u++) {
    uint32_t j = (uint32_t)(u % k);
    if (u >= k) {
      if (flip[j] == 0) { cf[j]++; str[j][0] = (uint8_t)((cf[j] * 7 + 101 * j + salt) % 249); }
      else { cl[j]++; str[j][15] = (uint8_t)((cl[j] * 11 + 59 * j + salt) % 249); }
      flip[j] ^= 1;
    }
    ob_put(&o, (const char *)str[j], 16);
    uint8_t sep = (uint8_t)(249 + (u % 7));
    ob_put(&o, (const char *)&sep, 1);
  }
  return 0;
}

int gg_random(uint64_t seed, uint8_t *dst, uint64_t n) {
  rng_t r; rng_seed(&r, seed);
  for (uint64_t i = 0; i < n; i += 8) {
    uint64_t x = rng_next(&r);
    for (int b = 0; b < 8 && i + b < n; b++) dst[i + b] = (uint8_t)(x >> (8 * b));
  }
  return 0;
}
