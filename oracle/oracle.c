/*
 * oracle.c — TEST INFRASTRUCTURE ONLY. A plain, slow, single-threaded CPU implementation of what the
 * Gompresso decompression hot path computes, written from the paper (PAPER.md, arXiv 1606.00519) and
 * FORMAT.md. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load it. It shares no code, header, table or constant generator with paper_1606_00519_b200/ (the product);
 * the two are written independently against FORMAT.md.
 *
 * Contents (citation = PAPER.md line numbers, "R<n>" = reading listed in DESIGN.md §3):
 *   or_compress        greedy exhaustive longest-match LZ77 per block (Fig. example), optional
 *                      Dependency Elimination (Fig. alg:dedeflate P:256-284, reading R4/R5), Byte or Bit
 *                      output. Bit: package-merge length-limited Huffman (CWL, R14),
 *                      canonical codes (RFC 1951 §3.2.2), DEFLATE symbols (R15).
 *   or_decompress      the plain definition: sequential expansion of the file's sequences (P:89-94,
 *                      P:767-779). Bit streams are decoded BIT BY BIT with the canonical count/first-code
 *                      walk (no lookup table), straight through all sub-blocks, checking the sub-block table.
 *   or_mrr_simulate    lock-step model of Multi-Round Resolution (Fig. alg:mrr P:174-193, prose P:196-253,
 *                      HWM reading R1, ready rule R4): per-group round counts and bytes per round.
 *   or_verify_de       the DE rule of FORMAT.md §4 on every group.
 *   or_package_merge / or_canonical_codes / or_parse_block: exposed for the pins in tests/.
 *
 * Parity pins (tests/test_oracle_*.py): round trip, RFC 1951 §3.2.2 worked example, stock zlib raw inflate of
 * the Bit symbol layer, Kraft equality and brute-force optimality of package-merge, brute-force greedy-parse
 * optimality on tiny inputs, the paper's LZ77 example, the MRR examples,
 * the nesting-depth point masses.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* status codes (same numeric meaning as include/gomp.h; FORMAT.md / DESIGN.md define them) */
enum {
  OR_OK = 0, OR_INVALID_ARG = -1, OR_BAD_MAGIC = -2, OR_UNSUPPORTED_VERSION = -3, OR_TRUNCATED = -4,
  OR_HEADER_INCONSISTENT = -5, OR_CORRUPT_STREAM = -6, OR_MALFORMED_BACKREF = -7, OR_NO_PROGRESS = -8,
  OR_DST_TOO_SMALL = -9
};

typedef struct {
  uint32_t mode;                 /* 0 Byte, 1 Bit */
  uint32_t de;                   /* Dependency Elimination on/off */
  uint32_t block_size;
  uint32_t window_size;
  uint32_t min_match;
  uint32_t max_match;
  uint32_t sub_block_seqs;       /* S; 0 = use sub_blocks_per_block */
  uint32_t sub_blocks_per_block;
  uint32_t cwl;
  uint32_t de_group;             /* sequences per DE group (warpHWM update period); 0 = 32 (the paper's warp) */
} or_params;

/* ------------------------------------------------------------------ little-endian helpers */
static uint32_t rd32(const uint8_t *p) { return (uint32_t)p[0] | (uint32_t)p[1] << 8 | (uint32_t)p[2] << 16 | (uint32_t)p[3] << 24; }
static uint64_t rd64(const uint8_t *p) { return (uint64_t)rd32(p) | (uint64_t)rd32(p + 4) << 32; }
static void wr32(uint8_t *p, uint32_t v) { for (int i = 0; i < 4; i++) p[i] = (uint8_t)(v >> (8 * i)); }
static void wr64(uint8_t *p, uint64_t v) { wr32(p, (uint32_t)v); wr32(p + 4, (uint32_t)(v >> 32)); }
static uint64_t align16(uint64_t x) { return (x + 15) & ~(uint64_t)15; }

/* ------------------------------------------------------------------ sequences */
typedef struct { uint32_t lit_len, L, dist; } seq_t;   /* L = 0: no back-reference */
typedef struct { seq_t *v; uint32_t n, cap; } seqvec;
static void sv_push(seqvec *s, uint32_t lit, uint32_t L, uint32_t dist) {
  if (s->n == s->cap) { s->cap = s->cap ? 2 * s->cap : 64; s->v = (seq_t *)realloc(s->v, sizeof(seq_t) * s->cap); }
  s->v[s->n].lit_len = lit; s->v[s->n].L = L; s->v[s->n].dist = dist; s->n++;
}

/*
 * Greedy parse of one block (src[0..n)), FORMAT.md §2 and DESIGN.md R2/R4/R5/R7/R10.
 * At cursor c every candidate source s with 1 <= c-s <= window, s >= 0 is tried; its length is the common
 * prefix capped by max_match, by n-c (block end) and by c-s (no overlap, R2). With DE (Fig. alg:dedeflate),
 * a candidate is admissible iff s >= ls (inside the pending literal string) or s < warpHWM, in which case its
 * length is also capped by warpHWM - s (R4/R5). The longest admissible candidate wins, ties to the smallest
 * distance (R7). warpHWM <- c after every 32nd emitted sequence (line alg:deupdate), or after every
 * de_group-th sequence for the wide DE groups of FORMAT.md §4 (P:82-85 gives the group size
 * as the warp width, a Kepler synchronisation choice).
 */
static void parse_block(const uint8_t *src, uint32_t n, const or_params *p, seqvec *out) {
  const uint32_t G = p->de_group ? p->de_group : 32;
  uint32_t c = 0, ls = 0, nseq = 0, hwm = 0;
  while (c < n) {
    uint32_t best_len = 0, best_dist = 0;
    uint32_t lo = c > p->window_size ? c - p->window_size : 0;
    for (uint32_t s = c; s-- > lo;) {            /* s = c-1 down to lo: increasing distance */
      uint32_t cap = p->max_match;
      if (n - c < cap) cap = n - c;
      if (c - s < cap) cap = c - s;
      if (p->de && s < ls) {
        if (s >= hwm) continue;                  /* source in [warpHWM, ls): inadmissible */
        if (hwm - s < cap) cap = hwm - s;
      }
      uint32_t len = 0;
      while (len < cap && src[s + len] == src[c + len]) len++;
      if (len > best_len) { best_len = len; best_dist = c - s; }
    }
    if (best_len >= p->min_match) {
      sv_push(out, c - ls, best_len, best_dist);
      c += best_len; ls = c; nseq++;
      if (nseq % G == 0) hwm = c;
    } else {
      c++;
      if (c - ls == 1023) {                      /* R10: close the run at 1023 literals */
        sv_push(out, 1023, 0, 0);
        ls = c; nseq++;
        if (nseq % G == 0) hwm = c;
      }
    }
  }
  if (c > ls) sv_push(out, c - ls, 0, 0);        /* final literal-only sequence */
}

/* ------------------------------------------------------------------ Huffman: package-merge (R14) */
typedef struct { uint64_t w; uint16_t *cnt; } pm_item;

/*
 * Length-limited Huffman code lengths by package-merge (Larmore & Hirschberg coin collector). Leaves are the
 * used symbols sorted by (frequency, symbol). Repeat maxlen-1 times: list <- merge(leaves, pairs(list)),
 * leaves first on equal weight. The first 2m-2 items of the final list select the code lengths: a symbol's
 * length is the number of selected items containing it. m = 1 -> length 1; m = 0 -> all zero.
 */
int or_package_merge(const uint64_t *freq, int n, int maxlen, uint8_t *lens) {
  int m = 0;
  int *sym = (int *)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
  for (int i = 0; i < n; i++) { lens[i] = 0; if (freq[i]) sym[m++] = i; }
  if (m == 0) { free(sym); return 0; }
  if (m == 1) { lens[sym[0]] = 1; free(sym); return 0; }
  if ((1 << maxlen) < m) { free(sym); return OR_INVALID_ARG; }
  for (int i = 1; i < m; i++)                      /* insertion sort by (freq, symbol) */
    for (int j = i; j > 0; j--) {
      int a = sym[j - 1], b = sym[j];
      if (freq[a] > freq[b] || (freq[a] == freq[b] && a > b)) { sym[j - 1] = b; sym[j] = a; } else break;
    }
  pm_item *leaves = (pm_item *)malloc(sizeof(pm_item) * (size_t)m);
  for (int i = 0; i < m; i++) {
    leaves[i].w = freq[sym[i]];
    leaves[i].cnt = (uint16_t *)calloc((size_t)n, sizeof(uint16_t));
    leaves[i].cnt[sym[i]] = 1;
  }
  int len = m;
  pm_item *list = (pm_item *)malloc(sizeof(pm_item) * (size_t)m);
  for (int i = 0; i < m; i++) { list[i].w = leaves[i].w; list[i].cnt = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)n); memcpy(list[i].cnt, leaves[i].cnt, sizeof(uint16_t) * (size_t)n); }
  for (int level = 1; level < maxlen; level++) {
    int np = len / 2;
    pm_item *pk = (pm_item *)malloc(sizeof(pm_item) * (size_t)(np > 0 ? np : 1));
    for (int i = 0; i < np; i++) {
      pk[i].w = list[2 * i].w + list[2 * i + 1].w;
      pk[i].cnt = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)n);
      for (int s = 0; s < n; s++) pk[i].cnt[s] = (uint16_t)(list[2 * i].cnt[s] + list[2 * i + 1].cnt[s]);
    }
    for (int i = 0; i < len; i++) free(list[i].cnt);
    free(list);
    list = (pm_item *)malloc(sizeof(pm_item) * (size_t)(m + np));
    int a = 0, b = 0, k = 0;
    while (a < m || b < np) {
      int take_leaf = (b >= np) || (a < m && leaves[a].w <= pk[b].w);
      if (take_leaf) {
        list[k].w = leaves[a].w;
        list[k].cnt = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)n);
        memcpy(list[k].cnt, leaves[a].cnt, sizeof(uint16_t) * (size_t)n);
        a++;
      } else {
        list[k] = pk[b];
        b++;
      }
      k++;
    }
    free(pk);
    len = k;
  }
  for (int i = 0; i < 2 * m - 2; i++)
    for (int s = 0; s < n; s++) lens[s] = (uint8_t)(lens[s] + list[i].cnt[s]);
  for (int i = 0; i < len; i++) free(list[i].cnt);
  free(list);
  for (int i = 0; i < m; i++) free(leaves[i].cnt);
  free(leaves);
  free(sym);
  return 0;
}

/* Canonical codes, RFC 1951 §3.2.2 steps 1-3 (codes are MSB-first integers of `len` bits). */
int or_canonical_codes(const uint8_t *lens, int n, uint32_t *codes) {
  uint32_t bl_count[16] = {0}, next_code[16] = {0};
  for (int i = 0; i < n; i++) { if (lens[i] > 15) return OR_INVALID_ARG; bl_count[lens[i]]++; }
  bl_count[0] = 0;
  uint32_t code = 0;
  for (int bits = 1; bits <= 15; bits++) { code = (code + bl_count[bits - 1]) << 1; next_code[bits] = code; }
  for (int i = 0; i < n; i++) { codes[i] = 0; if (lens[i]) codes[i] = next_code[lens[i]]++; }
  return 0;
}

/* ------------------------------------------------------------------ DEFLATE symbol tables, RFC 1951 §3.2.5 */
static const uint16_t LEN_BASE[29] = {3, 4, 5, 6, 7, 8, 9, 10, 11, 13, 15, 17, 19, 23, 27, 31,
                                      35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
static const uint8_t LEN_EXTRA[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 2,
                                      3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
static const uint16_t DIST_BASE[30] = {1, 2, 3, 4, 5, 7, 9, 13, 17, 25, 33, 49, 65, 97, 129, 193, 257, 385,
                                       513, 769, 1025, 1537, 2049, 3073, 4097, 6145, 8193, 12289, 16385, 24577};
static const uint8_t DIST_EXTRA[30] = {0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7,
                                       8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};

static int len_symbol(uint32_t L) {                 /* 257 + index of the code covering L */
  for (int i = 28; i >= 0; i--) if (L >= LEN_BASE[i]) { if (i == 28 && L != 258) continue; return i; }
  return -1;
}
static int dist_symbol(uint32_t d) {
  for (int i = 29; i >= 0; i--) if (d >= DIST_BASE[i]) return i;
  return -1;
}

/* ------------------------------------------------------------------ LSB-first bit writer (RFC 1951 §3.1.1) */
typedef struct { uint8_t *p; uint64_t nbits, cap_bits; } bitw;
static void bw_put(bitw *w, uint32_t value, int nbits) {           /* integer, LSB first */
  for (int i = 0; i < nbits; i++) {
    uint64_t pos = w->nbits++;
    if (pos >= w->cap_bits) continue;
    if ((value >> i) & 1u) w->p[pos >> 3] |= (uint8_t)(1u << (pos & 7));
  }
}
static void bw_code(bitw *w, uint32_t code, int len) {             /* Huffman code, MSB of the code first */
  for (int i = len - 1; i >= 0; i--) bw_put(w, (code >> i) & 1u, 1);
}

/* ------------------------------------------------------------------ compressor */
uint64_t or_compress_bound(uint64_t n, const or_params *p) {
  uint64_t nb = p->block_size ? (n + p->block_size - 1) / p->block_size : 0;
  /* worst case per block: every byte literal in 1023-runs; Bit adds trees + raw-ish symbols */
  uint64_t per_block = (uint64_t)p->block_size * 3 + 512;
  uint64_t subs = (uint64_t)p->block_size + 1;
  return 64 + nb * (32 + 8 * subs + per_block) + 64;
}

int or_compress(const uint8_t *src, uint64_t n, const or_params *p, uint8_t *dst, uint64_t cap, uint64_t *out_len) {
  if (!p || p->block_size < 16 || p->block_size % 16 || p->window_size < 1 || p->window_size > 32768 ||
      (p->min_match != 3 && p->min_match != 4) || p->max_match < p->min_match ||
      p->max_match > p->min_match + 62 || p->mode > 1 ||
      (p->mode == 1 && (p->cwl < 9 || p->cwl > 15 || (p->sub_block_seqs == 0 && p->sub_blocks_per_block == 0))) ||
      p->de_group % 32 || p->de_group > 224)
    return OR_INVALID_ARG;
  uint32_t nb = (uint32_t)((n + p->block_size - 1) / p->block_size);
  seqvec *seqs = (seqvec *)calloc(nb ? nb : 1, sizeof(seqvec));
  uint32_t *S = (uint32_t *)calloc(nb ? nb : 1, sizeof(uint32_t));
  uint32_t *nsub = (uint32_t *)calloc(nb ? nb : 1, sizeof(uint32_t));
  uint64_t n_sub_total = 0;
  for (uint32_t b = 0; b < nb; b++) {
    uint64_t off = (uint64_t)b * p->block_size;
    uint32_t len = (uint32_t)((n - off) < p->block_size ? (n - off) : p->block_size);
    parse_block(src + off, len, p, &seqs[b]);
    if (p->mode == 1) {
      uint32_t ns = seqs[b].n;
      S[b] = p->sub_block_seqs ? p->sub_block_seqs : (ns + p->sub_blocks_per_block - 1) / p->sub_blocks_per_block;
      if (S[b] == 0) S[b] = 1;
      nsub[b] = (ns + S[b] - 1) / S[b];
      n_sub_total += nsub[b];
    }
  }
  uint64_t payload_base = align16(64 + 32ull * nb + 8ull * n_sub_total);
  if (cap < payload_base + 16) { free(seqs); free(S); free(nsub); return OR_DST_TOO_SMALL; }
  memset(dst, 0, cap < payload_base ? cap : payload_base);
  uint64_t pos = payload_base;
  uint32_t sub_at = 0, max_tokens = 0;
  for (uint32_t b = 0; b < nb; b++) {
    uint64_t off = (uint64_t)b * p->block_size;
    const uint8_t *blk = src + off;
    seqvec *sv = &seqs[b];
    uint32_t n_lit = 0;
    for (uint32_t i = 0; i < sv->n; i++) n_lit += sv->v[i].lit_len;
    uint8_t *ent = dst + 64 + 32ull * b;
    uint64_t start = pos;
    if (p->mode == 0) {
      uint64_t need = align16(4ull * sv->n + n_lit);
      if (pos + need + 16 > cap) { free(seqs); free(S); free(nsub); return OR_DST_TOO_SMALL; }
      memset(dst + pos, 0, need);
      uint32_t c = 0, lp = 0;
      uint8_t *lits = dst + pos + 4ull * sv->n;
      for (uint32_t i = 0; i < sv->n; i++) {
        seq_t q = sv->v[i];
        uint32_t mcode = q.L ? q.L - p->min_match + 1 : 0;
        uint32_t rec = q.lit_len | mcode << 10 | (q.L ? (q.dist - 1) << 16 : 0);
        wr32(dst + pos + 4ull * i, rec);
        memcpy(lits + lp, blk + c, q.lit_len);
        lp += q.lit_len;
        c += q.lit_len + q.L;
      }
      pos += need;
    } else {
      /* symbol frequencies of the block ("both trees are created from the token frequencies") */
      uint64_t flit[286] = {0}, fdist[30] = {0};
      uint32_t c = 0;
      for (uint32_t i = 0; i < sv->n; i++) {
        seq_t q = sv->v[i];
        for (uint32_t k = 0; k < q.lit_len; k++) flit[blk[c + k]]++;
        if (q.L) { flit[257 + len_symbol(q.L)]++; fdist[dist_symbol(q.dist)]++; }
        c += q.lit_len + q.L;
      }
      flit[256]++;
      uint8_t llen[286], dlen[30];
      uint32_t lcode[286], dcode[30];
      if (or_package_merge(flit, 286, (int)p->cwl, llen) || or_package_merge(fdist, 30, (int)p->cwl, dlen)) {
        free(seqs); free(S); free(nsub); return OR_INVALID_ARG;
      }
      int any_d = 0;
      for (int i = 0; i < 30; i++) any_d |= dlen[i] != 0;
      if (!any_d) dlen[0] = 1;                      /* R14: one dummy distance code */
      or_canonical_codes(llen, 286, lcode);
      or_canonical_codes(dlen, 30, dcode);
      uint64_t room = cap - pos;
      if (room < 160 + 16) { free(seqs); free(S); free(nsub); return OR_DST_TOO_SMALL; }
      memset(dst + pos, 0, room > (uint64_t)p->block_size * 3 + 512 ? (uint64_t)p->block_size * 3 + 512 : room);
      for (int i = 0; i < 286; i++) dst[pos + i / 2] |= (uint8_t)(llen[i] << (4 * (i & 1)));
      for (int i = 0; i < 30; i++) dst[pos + 143 + i / 2] |= (uint8_t)(dlen[i] << (4 * (i & 1)));
      bitw w = {dst + pos + 160, 0, (room - 160 - 16) * 8};
      uint32_t k = 0, S_b = S[b];
      c = 0;
      for (uint32_t sb = 0; sb < nsub[b]; sb++) {
        uint64_t bit0 = w.nbits;
        uint32_t sub_lit = 0;
        uint32_t end = (sb + 1) * S_b < sv->n ? (sb + 1) * S_b : sv->n;
        for (; k < end; k++) {
          seq_t q = sv->v[k];
          for (uint32_t t = 0; t < q.lit_len; t++) bw_code(&w, lcode[blk[c + t]], llen[blk[c + t]]);
          sub_lit += q.lit_len;
          if (q.L) {
            int li = len_symbol(q.L), di = dist_symbol(q.dist);
            bw_code(&w, lcode[257 + li], llen[257 + li]);
            bw_put(&w, q.L - LEN_BASE[li], LEN_EXTRA[li]);
            bw_code(&w, dcode[di], dlen[di]);
            bw_put(&w, q.dist - DIST_BASE[di], DIST_EXTRA[di]);
          }
          c += q.lit_len + q.L;
        }
        if (sb + 1 == nsub[b]) bw_code(&w, lcode[256], llen[256]);   /* EOB ends the block */
        uint8_t *se = dst + payload_base - 0;                          /* placeholder, set below */
        (void)se;
        uint8_t *sent = dst + 64 + 32ull * nb + 8ull * (sub_at + sb);
        wr32(sent, (uint32_t)(w.nbits - bit0));
        wr32(sent + 4, sub_lit);
      }
      if (w.nbits > w.cap_bits) { free(seqs); free(S); free(nsub); return OR_DST_TOO_SMALL; }
      pos += align16(160 + (w.nbits + 7) / 8);
      uint32_t tok = 4 * sv->n + n_lit;
      if (tok > max_tokens) max_tokens = tok;
    }
    wr64(ent, start);
    wr32(ent + 8, (uint32_t)(pos - start));
    wr32(ent + 12, sv->n);
    wr32(ent + 16, n_lit);
    wr32(ent + 20, p->mode ? sub_at : 0);
    wr32(ent + 24, p->mode ? S[b] : 0);
    wr32(ent + 28, p->mode ? nsub[b] : 0);
    sub_at += p->mode ? nsub[b] : 0;
  }
  if (pos + 16 > cap) { free(seqs); free(S); free(nsub); return OR_DST_TOO_SMALL; }
  memset(dst + pos, 0, 16);
  pos += 16;
  uint8_t *h = dst;
  memcpy(h, "GMPR", 4);
  h[4] = 1; h[5] = (uint8_t)p->mode; h[6] = (uint8_t)(p->de ? 1 : 0);
  h[7] = (uint8_t)p->min_match; h[8] = (uint8_t)p->max_match; h[9] = (uint8_t)(p->mode ? p->cwl : 0);
  h[10] = (uint8_t)(p->de_group ? p->de_group : 32); h[11] = 0;
  wr32(h + 12, p->block_size); wr32(h + 16, p->window_size); wr32(h + 20, nb);
  wr64(h + 24, n); wr64(h + 32, pos);
  wr32(h + 40, (uint32_t)n_sub_total); wr32(h + 44, p->mode ? max_tokens : 0);
  wr64(h + 48, payload_base); wr32(h + 56, 0); wr32(h + 60, 0);
  *out_len = pos;
  for (uint32_t b = 0; b < nb; b++) free(seqs[b].v);
  free(seqs); free(S); free(nsub);
  return OR_OK;
}

/* ------------------------------------------------------------------ reader */
typedef struct {
  uint32_t mode, de, min_match, max_match, cwl, block_size, window, nb, n_sub_total, max_tokens, de_group;
  uint64_t total, file_len, payload_base;
} or_hdr;

static int read_header(const uint8_t *f, uint64_t len, or_hdr *h) {
  if (len < 64) return OR_TRUNCATED;
  if (memcmp(f, "GMPR", 4)) return OR_BAD_MAGIC;
  if (f[4] != 1) return OR_UNSUPPORTED_VERSION;
  h->mode = f[5]; h->de = f[6] & 1; h->min_match = f[7]; h->max_match = f[8]; h->cwl = f[9];
  h->block_size = rd32(f + 12); h->window = rd32(f + 16); h->nb = rd32(f + 20);
  h->total = rd64(f + 24); h->file_len = rd64(f + 32); h->n_sub_total = rd32(f + 40);
  h->max_tokens = rd32(f + 44); h->payload_base = rd64(f + 48); h->de_group = f[10];
  if (h->mode > 1 || (f[6] & ~1u) || f[10] == 0 || f[10] % 32 || f[11] || rd32(f + 56) || rd32(f + 60))
    return OR_HEADER_INCONSISTENT;
  if (h->min_match != 3 && h->min_match != 4) return OR_HEADER_INCONSISTENT;
  if (h->max_match < h->min_match || h->max_match > h->min_match + 62) return OR_HEADER_INCONSISTENT;
  if (h->block_size < 16 || h->block_size % 16 || h->window < 1 || h->window > 32768) return OR_HEADER_INCONSISTENT;
  if (h->mode == 1 && (h->cwl < 9 || h->cwl > 15)) return OR_HEADER_INCONSISTENT;
  if (h->mode == 0 && (h->cwl || h->n_sub_total || h->max_tokens)) return OR_HEADER_INCONSISTENT;
  if ((uint64_t)h->nb != (h->total + h->block_size - 1) / h->block_size) return OR_HEADER_INCONSISTENT;
  if (h->payload_base != align16(64 + 32ull * h->nb + 8ull * h->n_sub_total)) return OR_HEADER_INCONSISTENT;
  if (h->file_len > len) return OR_TRUNCATED;
  if (h->file_len < h->payload_base + 16) return OR_HEADER_INCONSISTENT;
  return OR_OK;
}

typedef struct { uint64_t off; uint32_t plen, n_seq, n_lit, sub_first, S, n_sub; } or_blk;

static int read_block(const uint8_t *f, const or_hdr *h, uint32_t b, or_blk *e) {
  const uint8_t *p = f + 64 + 32ull * b;
  e->off = rd64(p); e->plen = rd32(p + 8); e->n_seq = rd32(p + 12); e->n_lit = rd32(p + 16);
  e->sub_first = rd32(p + 20); e->S = rd32(p + 24); e->n_sub = rd32(p + 28);
  if (e->off % 16 || e->plen % 16 || e->off < h->payload_base || e->off + e->plen > h->file_len - 16) return OR_HEADER_INCONSISTENT;
  if (h->mode == 0) {
    if (e->sub_first || e->S || e->n_sub) return OR_HEADER_INCONSISTENT;
    if (4ull * e->n_seq + e->n_lit > e->plen) return OR_HEADER_INCONSISTENT;
  } else {
    if (e->S == 0 || e->n_sub != (e->n_seq + e->S - 1) / e->S) return OR_HEADER_INCONSISTENT;
    if ((uint64_t)e->sub_first + e->n_sub > h->n_sub_total || e->plen < 160) return OR_HEADER_INCONSISTENT;
    if (4ull * e->n_seq + e->n_lit > h->max_tokens) return OR_HEADER_INCONSISTENT;
  }
  return OR_OK;
}

/* bit-by-bit canonical decoder (RFC 1951 §3.2.2 counts/first codes; no table lookup) */
typedef struct { uint16_t count[16]; uint16_t sym[288]; int nsym; } canon;
static int canon_build(const uint8_t *lens, int n, canon *c) {
  memset(c, 0, sizeof(*c));
  for (int i = 0; i < n; i++) c->count[lens[i]]++;
  c->count[0] = 0;
  int left = 1;                                   /* Kraft: over-subscribed sets are invalid */
  for (int l = 1; l <= 15; l++) { left <<= 1; left -= c->count[l]; if (left < 0) return OR_CORRUPT_STREAM; }
  int offs[16]; offs[1] = 0;
  for (int l = 1; l < 15; l++) offs[l + 1] = offs[l] + c->count[l];
  for (int i = 0; i < n; i++) if (lens[i]) c->sym[offs[lens[i]]++] = (uint16_t)i;
  c->nsym = n;
  return OR_OK;
}
typedef struct { const uint8_t *p; uint64_t pos, end; } bitr;
static int br_bit(bitr *r) {
  if (r->pos >= r->end) { r->pos++; return 0; }
  int b = (r->p[r->pos >> 3] >> (r->pos & 7)) & 1;
  r->pos++;
  return b;
}
static uint32_t br_bits(bitr *r, int n) { uint32_t v = 0; for (int i = 0; i < n; i++) v |= (uint32_t)br_bit(r) << i; return v; }
static int canon_decode(bitr *r, const canon *c) {
  int code = 0, first = 0, index = 0;
  for (int l = 1; l <= 15; l++) {
    code |= br_bit(r);
    int count = c->count[l];
    if (code - first < count) return c->sym[index + (code - first)];
    index += count; first += count; first <<= 1; code <<= 1;
  }
  return -1;
}

/*
 * Decode block b into its sequence list (Byte: read records; Bit: bit-by-bit decode of all sub-blocks in
 * order, checking each sub-block's sequence count, literal count and bit size against the table, R13/R16).
 * lits receives the block's literal bytes (n_lit).
 */
static int block_sequences(const uint8_t *f, const or_hdr *h, const or_blk *e, uint32_t b, seqvec *out, uint8_t *lits) {
  const uint8_t *pl = f + e->off;
  if (h->mode == 0) {
    for (uint32_t i = 0; i < e->n_seq; i++) {
      uint32_t r = rd32(pl + 4ull * i);
      uint32_t lit = r & 1023, mcode = (r >> 10) & 63, dist = (r >> 16) + 1;
      uint32_t L = mcode ? mcode + h->min_match - 1 : 0;
      if (!mcode && (r >> 16)) return OR_CORRUPT_STREAM;
      sv_push(out, lit, L, L ? dist : 0);
    }
    memcpy(lits, pl + 4ull * e->n_seq, e->n_lit);
    return OR_OK;
  }
  uint8_t llen[286], dlen[30];
  for (int i = 0; i < 286; i++) llen[i] = (pl[i / 2] >> (4 * (i & 1))) & 15;
  for (int i = 0; i < 30; i++) dlen[i] = (pl[143 + i / 2] >> (4 * (i & 1))) & 15;
  for (int i = 0; i < 286; i++) if (llen[i] > h->cwl) return OR_CORRUPT_STREAM;
  for (int i = 0; i < 30; i++) if (dlen[i] > h->cwl) return OR_CORRUPT_STREAM;
  if (pl[158] || pl[159]) return OR_CORRUPT_STREAM;
  canon cl, cd;
  if (canon_build(llen, 286, &cl) || canon_build(dlen, 30, &cd)) return OR_CORRUPT_STREAM;
  bitr r = {pl + 160, 0, (uint64_t)(e->plen - 160) * 8};
  uint32_t nl = 0;
  uint32_t lit = 0;
  for (uint32_t sb = 0; sb < e->n_sub; sb++) {
    const uint8_t *se = f + 64 + 32ull * h->nb + 8ull * (e->sub_first + sb);
    uint32_t bit_size = rd32(se), sub_nlit = rd32(se + 4);
    uint64_t bit0 = r.pos;
    uint32_t seq_end = (sb + 1) * e->S < e->n_seq ? (sb + 1) * e->S : e->n_seq;
    int last = sb + 1 == e->n_sub;
    uint32_t lit0 = nl;
    for (;;) {
      if (!last && out->n == seq_end) break;
      int s = canon_decode(&r, &cl);
      if (s < 0 || r.pos > r.end) return OR_CORRUPT_STREAM;
      if (s < 256) {
        if (nl >= e->n_lit) return OR_CORRUPT_STREAM;
        lits[nl++] = (uint8_t)s;
        if (++lit == 1023) { sv_push(out, 1023, 0, 0); lit = 0; }
      } else if (s == 256) {
        if (!last) return OR_CORRUPT_STREAM;
        if (lit) { sv_push(out, lit, 0, 0); lit = 0; }
        break;
      } else {
        int li = s - 257;
        if (li > 28) return OR_CORRUPT_STREAM;
        uint32_t L = LEN_BASE[li] + br_bits(&r, LEN_EXTRA[li]);
        int ds = canon_decode(&r, &cd);
        if (ds < 0 || ds > 29) return OR_CORRUPT_STREAM;
        uint32_t dist = DIST_BASE[ds] + br_bits(&r, DIST_EXTRA[ds]);
        if (L < h->min_match || L > h->max_match) return OR_CORRUPT_STREAM;
        if (r.pos > r.end) return OR_CORRUPT_STREAM;
        sv_push(out, lit, L, dist);
        lit = 0;
      }
      if (out->n > seq_end) return OR_CORRUPT_STREAM;
    }
    if (out->n != seq_end || lit) return OR_CORRUPT_STREAM;
    if (r.pos - bit0 != bit_size || nl - lit0 != sub_nlit) return OR_CORRUPT_STREAM;
  }
  (void)b;
  if (out->n != e->n_seq || nl != e->n_lit) return OR_CORRUPT_STREAM;
  return OR_OK;
}

/* sequential expansion (the definition) with the FORMAT.md §2 checks */
static int expand(const or_hdr *h, const seqvec *sv, const uint8_t *lits, uint32_t n_lit, uint8_t *out, uint32_t ulen) {
  uint64_t o = 0, lp = 0;
  for (uint32_t i = 0; i < sv->n; i++) {
    seq_t q = sv->v[i];
    if (q.lit_len > 1023) return OR_CORRUPT_STREAM;
    if (lp + q.lit_len > n_lit || o + q.lit_len > ulen) return OR_CORRUPT_STREAM;
    for (uint32_t k = 0; k < q.lit_len; k++) out[o++] = lits[lp++];
    if (q.L) {
      if (q.dist < q.L || q.dist < 1 || q.dist > h->window || q.dist > o) return OR_MALFORMED_BACKREF;
      if (q.L < h->min_match || q.L > h->max_match) return OR_MALFORMED_BACKREF;
      if (o + q.L > ulen) return OR_CORRUPT_STREAM;
      for (uint32_t k = 0; k < q.L; k++) { out[o] = out[o - q.dist]; o++; }
    }
  }
  if (o != ulen || lp != n_lit) return OR_CORRUPT_STREAM;
  return OR_OK;
}

static uint32_t block_ulen(const or_hdr *h, uint32_t b) {
  uint64_t off = (uint64_t)b * h->block_size;
  return (uint32_t)((h->total - off) < h->block_size ? (h->total - off) : h->block_size);
}

int or_info(const uint8_t *f, uint64_t len, uint64_t *total, uint32_t *nb) {
  or_hdr h;
  int st = read_header(f, len, &h);
  if (st) return st;
  *total = h.total; *nb = h.nb;
  return OR_OK;
}

/* decompress blocks [b0, b1) into dst (dst[0] = first byte of block b0) */
int or_decompress_range(const uint8_t *f, uint64_t len, uint32_t b0, uint32_t b1, uint8_t *dst, uint64_t cap, uint32_t *err_block) {
  or_hdr h;
  int st = read_header(f, len, &h);
  *err_block = 0;
  if (st) return st;
  if (b1 > h.nb || b0 > b1) return OR_INVALID_ARG;
  uint64_t need = 0;
  for (uint32_t b = b0; b < b1; b++) need += block_ulen(&h, b);
  if (cap < need) return OR_DST_TOO_SMALL;
  uint8_t *lits = (uint8_t *)malloc((size_t)h.block_size * 4 + 16);
  uint64_t o = 0;
  for (uint32_t b = b0; b < b1; b++) {
    or_blk e;
    seqvec sv = {0, 0, 0};
    *err_block = b;
    st = read_block(f, &h, b, &e);
    if (!st && e.n_lit > h.block_size) st = OR_HEADER_INCONSISTENT;
    if (!st) st = block_sequences(f, &h, &e, b, &sv, lits);
    if (!st) st = expand(&h, &sv, lits, e.n_lit, dst + o, block_ulen(&h, b));
    free(sv.v);
    if (st) { free(lits); return st; }
    o += block_ulen(&h, b);
  }
  free(lits);
  *err_block = 0;
  return OR_OK;
}

int or_decompress(const uint8_t *f, uint64_t len, uint8_t *dst, uint64_t cap, uint64_t *out_len, uint32_t *err_block) {
  or_hdr h;
  int st = read_header(f, len, &h);
  *err_block = 0;
  if (st) return st;
  st = or_decompress_range(f, len, 0, h.nb, dst, cap, err_block);
  if (!st) *out_len = h.total;
  return st;
}

/* sequence list of block b: arrays of n_seq entries (caller sizes them by the block table) */
int or_block_sequences(const uint8_t *f, uint64_t len, uint32_t b, uint32_t *lit_len, uint32_t *L, uint32_t *dist, uint32_t cap, uint32_t *n_out) {
  or_hdr h; or_blk e;
  int st = read_header(f, len, &h);
  if (st) return st;
  if (b >= h.nb) return OR_INVALID_ARG;
  if ((st = read_block(f, &h, b, &e))) return st;
  if (e.n_lit > h.block_size) return OR_HEADER_INCONSISTENT;
  seqvec sv = {0, 0, 0};
  uint8_t *lits = (uint8_t *)malloc((size_t)h.block_size + 16);
  st = block_sequences(f, &h, &e, b, &sv, lits);
  free(lits);
  if (!st && sv.n > cap) st = OR_DST_TOO_SMALL;
  if (!st) for (uint32_t i = 0; i < sv.n; i++) { lit_len[i] = sv.v[i].lit_len; L[i] = sv.v[i].L; dist[i] = sv.v[i].dist; }
  *n_out = sv.n;
  free(sv.v);
  return st;
}

/* parse of a raw block, exposed for the brute-force pins */
int or_parse_block(const uint8_t *src, uint32_t n, const or_params *p, uint32_t *lit_len, uint32_t *L, uint32_t *dist, uint32_t cap, uint32_t *n_out) {
  seqvec sv = {0, 0, 0};
  parse_block(src, n, p, &sv);
  int st = sv.n > cap ? OR_DST_TOO_SMALL : OR_OK;
  if (!st) for (uint32_t i = 0; i < sv.n; i++) { lit_len[i] = sv.v[i].lit_len; L[i] = sv.v[i].L; dist[i] = sv.v[i].dist; }
  *n_out = sv.n;
  free(sv.v);
  return st;
}

/*
 * MRR, lock-step model of Fig. alg:mrr for one 32-sequence group (lanes 0..n-1), R1/R3/R4/R19/R20.
 * dst_i = back-reference destination, ls_i = literal start, src_i = dst_i - dist_i (block-relative).
 * pending_i = (L_i > 0). Each round: HWM <- dst of the lowest pending lane (the end of the gap-free written
 * prefix); lane i is ready iff pending and (src_i + L_i <= HWM or src_i >= ls_i); all ready lanes copy;
 * they clear pending. Returns the number of rounds; bytes[r] accumulates the bytes copied in round r (1-based).
 */
static int mrr_group(const uint32_t *ls, const uint32_t *dst, const uint32_t *src, const uint32_t *L, int n, uint64_t *bytes) {
  int pending[32], rounds = 0;
  for (int i = 0; i < n; i++) pending[i] = L[i] > 0;
  for (;;) {
    int p = -1;
    for (int i = 0; i < n; i++) if (pending[i]) { p = i; break; }
    if (p < 0) break;
    uint32_t hwm = dst[p];
    int ready[32], any = 0;
    for (int i = 0; i < n; i++) {
      ready[i] = pending[i] && (src[i] + L[i] <= hwm || src[i] >= ls[i]);
      any |= ready[i];
    }
    if (!any) return -1;                         /* cannot happen on a valid file */
    rounds++;
    for (int i = 0; i < n; i++) if (ready[i]) { pending[i] = 0; if (bytes && rounds < 33) bytes[rounds] += L[i]; }
  }
  return rounds;
}

/* rounds histogram (hist[r] = groups needing r rounds, r = 0..32) and bytes per round over the whole file */
int or_mrr_simulate(const uint8_t *f, uint64_t len, uint64_t *hist, uint64_t *bytes) {
  or_hdr h;
  int st = read_header(f, len, &h);
  if (st) return st;
  for (int i = 0; i < 33; i++) { hist[i] = 0; bytes[i] = 0; }
  uint8_t *lits = (uint8_t *)malloc((size_t)h.block_size + 16);
  for (uint32_t b = 0; b < h.nb; b++) {
    or_blk e;
    seqvec sv = {0, 0, 0};
    if ((st = read_block(f, &h, b, &e)) || e.n_lit > h.block_size || (st = block_sequences(f, &h, &e, b, &sv, lits))) {
      free(sv.v); free(lits); return st ? st : OR_HEADER_INCONSISTENT;
    }
    uint32_t o = 0;
    for (uint32_t g = 0; g * 32 < sv.n; g++) {
      uint32_t ls[32], dst[32], src[32], L[32];
      int n = (int)(sv.n - g * 32 < 32 ? sv.n - g * 32 : 32);
      for (int i = 0; i < n; i++) {
        seq_t q = sv.v[g * 32 + i];
        ls[i] = o; dst[i] = o + q.lit_len; L[i] = q.L; src[i] = q.L ? dst[i] - q.dist : 0;
        o += q.lit_len + q.L;
      }
      int r = mrr_group(ls, dst, src, L, n, bytes);
      if (r < 0) { free(sv.v); free(lits); return OR_NO_PROGRESS; }
      hist[r]++;
    }
    free(sv.v);
  }
  free(lits);
  return OR_OK;
}

/* MRR on an explicit list of (lit_len, L, dist) for one group starting at block offset o0 (paper examples) */
int or_mrr_group_rounds(const uint32_t *lit_len, const uint32_t *L, const uint32_t *dist, int n, uint32_t o0,
                        uint64_t *bytes_per_round, uint32_t *round_of_lane) {
  uint32_t ls[32], dst[32], src[32], Ls[32];
  if (n < 0 || n > 32) return OR_INVALID_ARG;
  uint32_t o = o0;
  for (int i = 0; i < n; i++) { ls[i] = o; dst[i] = o + lit_len[i]; Ls[i] = L[i]; src[i] = L[i] ? dst[i] - dist[i] : 0; o += lit_len[i] + L[i]; }
  /* per-lane round numbers: rerun the model, recording when each lane copies */
  int pending[32], rounds = 0;
  for (int i = 0; i < n; i++) { pending[i] = Ls[i] > 0; round_of_lane[i] = 0; }
  for (int i = 0; i < 33; i++) bytes_per_round[i] = 0;
  for (;;) {
    int p = -1;
    for (int i = 0; i < n; i++) if (pending[i]) { p = i; break; }
    if (p < 0) break;
    uint32_t hwm = dst[p];
    int any = 0, ready[32];
    for (int i = 0; i < n; i++) { ready[i] = pending[i] && (src[i] + Ls[i] <= hwm || src[i] >= ls[i]); any |= ready[i]; }
    if (!any) return OR_NO_PROGRESS;
    rounds++;
    for (int i = 0; i < n; i++) if (ready[i]) { pending[i] = 0; round_of_lane[i] = (uint32_t)rounds; bytes_per_round[rounds] += Ls[i]; }
  }
  return rounds;
}

/* DE rule of FORMAT.md §4 on every group: returns 1 if it holds everywhere, 0 if not, <0 on a bad file */
int or_verify_de(const uint8_t *f, uint64_t len) {
  or_hdr h;
  int st = read_header(f, len, &h);
  if (st) return st;
  uint8_t *lits = (uint8_t *)malloc((size_t)h.block_size + 16);
  int ok = 1;
  for (uint32_t b = 0; b < h.nb && ok; b++) {
    or_blk e;
    seqvec sv = {0, 0, 0};
    if ((st = read_block(f, &h, b, &e)) || e.n_lit > h.block_size || (st = block_sequences(f, &h, &e, b, &sv, lits))) {
      free(sv.v); free(lits); return st ? st : OR_HEADER_INCONSISTENT;
    }
    uint32_t o = 0, H = 0;
    for (uint32_t i = 0; i < sv.n; i++) {
      if (i % h.de_group == 0) H = o;
      seq_t q = sv.v[i];
      uint32_t ls = o, d = o + q.lit_len;
      if (q.L) {
        uint32_t s = d - q.dist;
        if (!(s + q.L <= H || s >= ls)) ok = 0;
      }
      o += q.lit_len + q.L;
    }
    free(sv.v);
  }
  free(lits);
  return ok;
}
