// compress.cpp — host (CPU) Gompresso compressor: the producer of the decoder's input.
//
// Block-parallel over std::threads with a shared block counter (blocks are compressed "independently and in
// parallel"). Per block: greedy LZ77 with optional Dependency Elimination (Fig. alg:dedeflate,
// P:256-284; readings R4/R5/R7/R10 of DESIGN.md), then Byte records (R11) or Bit Huffman coding (two trees
// per block from the block's token frequencies; package-merge length limit CWL, R14;
// canonical codes; DEFLATE symbols, R15; sub-blocks with bit sizes, R12/R13).
//
// Match finders:
//   0 (default) hash chains over all earlier positions of the window, examined nearest first. With
//     max_chain = 0 every candidate whose first min_match bytes agree is examined, so the parse equals the
//     exhaustive greedy longest-match parse of FORMAT.md (tests check byte identity with the oracle's files).
//   1 the LZ4-style matcher the paper modified for DE: one table slot per trigram hash holding the
//     most recent position, replaced only if the stored position is more than min_staleness bytes behind.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <new>
#include <thread>
#include <vector>

#include "format.hpp"
#include "gomp.h"

namespace gomp {
namespace {

struct Seq {
  uint32_t lit, L, dist;
};

// ------------------------------------------------------------------ RFC 1951 §3.2.5 length / distance codes
constexpr uint16_t kLenBase[29] = {3,  4,  5,  6,  7,  8,  9,  10, 11,  13,  15,  17,  19,  23, 27,
                                   31, 35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
constexpr uint8_t kLenExtra[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
constexpr uint16_t kDistBase[30] = {1,    2,    3,    4,    5,    7,     9,     13,    17,  25,
                                    33,   49,   65,   97,   129,  193,   257,   385,   513, 769,
                                    1025, 1537, 2049, 3073, 4097, 6145, 8193, 12289, 16385, 24577};
constexpr uint8_t kDistExtra[30] = {0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};

inline int len_index(uint32_t L) {
  if (L == 258) return 28;
  int i = 27;
  while (kLenBase[i] > L) --i;
  return i;
}
inline int dist_index(uint32_t d) {
  int i = 29;
  while (kDistBase[i] > d) --i;
  return i;
}

// ------------------------------------------------------------------ greedy parse of one block
struct ParseScratch {
  std::vector<int32_t> head, prev;
};

inline uint32_t hash_at(const uint8_t* p, uint32_t mm, int bits) {
  uint32_t v = mm == 4 ? (uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24)
                       : (uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16);
  return (v * 2654435761u) >> (32 - bits);
}

void parse_block(const uint8_t* src, uint32_t n, const gomp_params& p, std::vector<Seq>& out, ParseScratch& s) {
  const uint32_t mm = p.min_match, win = p.window_size;
  const int hbits = p.match_finder == 1 ? 14 : 16;
  s.head.assign(size_t(1) << hbits, -1);
  if (p.match_finder == 0) s.prev.resize(n > 0 ? n : 1);
  uint32_t c = 0, ls = 0, nseq = 0, hwm = 0, ins = 0;
  const uint32_t G = p.de_group;
  auto emit = [&](uint32_t lit, uint32_t L, uint32_t d) {
    out.push_back({lit, L, d});
    if (++nseq % G == 0) hwm = c;  // warpHWM <- pos after every de_group (32) sequences
  };
  while (c < n) {
    // index every position < c that can start a min_match-byte match
    for (; ins < c; ++ins) {
      if (ins + mm > n) { ins = c; break; }
      uint32_t h = hash_at(src + ins, mm, hbits);
      if (p.match_finder == 0) {
        s.prev[ins] = s.head[h];
        s.head[h] = int32_t(ins);
      } else {
        int32_t old = s.head[h];
        if (old < 0 || ins - uint32_t(old) > p.min_staleness) s.head[h] = int32_t(ins);
      }
    }
    uint32_t best = 0, bdist = 0;
    const uint32_t maxL = std::min<uint32_t>(p.max_match, n - c);
    if (maxL >= mm) {
      int32_t cand = s.head[hash_at(src + c, mm, hbits)];
      uint32_t steps = 0;
      while (cand >= 0 && c - uint32_t(cand) <= win) {
        const uint32_t sp = uint32_t(cand);
        uint32_t cap = std::min(maxL, c - sp);  // no overlap (R2)
        bool admissible = true;
        if (p.de && sp < ls) {                   // DE (R4/R5): below warpHWM, truncated to it
          if (sp >= hwm) admissible = false;
          else cap = std::min(cap, hwm - sp);
        }
        if (admissible && cap > best && cap >= mm && src[sp + best] == src[c + best]) {
          uint32_t len = 0;
          while (len < cap && src[sp + len] == src[c + len]) ++len;
          if (len > best) {
            best = len;
            bdist = c - sp;
            if (best == maxL) break;
          }
        }
        if (p.match_finder == 1) break;
        if (p.max_chain && ++steps >= p.max_chain) break;
        cand = s.prev[sp];
      }
    }
    if (best >= mm) {
      const uint32_t lit = c - ls;
      c += best;
      emit(lit, best, bdist);
      ls = c;
    } else {
      ++c;
      if (c - ls == kMaxLitRun) {  // R10: close a literal run at 1023 bytes
        emit(kMaxLitRun, 0, 0);
        ls = c;
      }
    }
  }
  if (c > ls) emit(c - ls, 0, 0);
}

// ------------------------------------------------------------------ package-merge (R14)
// Leaves = used symbols sorted by (freq, symbol). lists[maxlen] = leaves; lists[d] = merge(leaves,
// pairs(lists[d+1])), a leaf before a package of equal weight. The first 2m-2 items of lists[1] are selected;
// a selected package selects the first 2P items of the next list. Length = times a symbol is selected.
void package_merge(const uint64_t* freq, int n, int maxlen, uint8_t* lens) {
  std::vector<int> sym;
  for (int i = 0; i < n; ++i) {
    lens[i] = 0;
    if (freq[i]) sym.push_back(i);
  }
  const int m = int(sym.size());
  if (m == 0) return;
  if (m == 1) { lens[sym[0]] = 1; return; }
  std::stable_sort(sym.begin(), sym.end(), [&](int a, int b) { return freq[a] < freq[b]; });
  struct Item { uint64_t w; int16_t sym; };  // sym < 0: package
  std::vector<std::vector<Item>> lists(size_t(maxlen) + 1);
  for (int i = 0; i < m; ++i) lists[maxlen].push_back({freq[sym[i]], int16_t(sym[i])});
  for (int d = maxlen - 1; d >= 1; --d) {
    const auto& prev = lists[d + 1];
    const size_t np = prev.size() / 2;
    auto& cur = lists[d];
    cur.reserve(m + np);
    size_t a = 0, b = 0;
    while (a < size_t(m) || b < np) {
      const uint64_t pw = b < np ? prev[2 * b].w + prev[2 * b + 1].w : 0;
      if (b >= np || (a < size_t(m) && freq[sym[a]] <= pw)) { cur.push_back({freq[sym[a]], int16_t(sym[a])}); ++a; }
      else { cur.push_back({pw, -1}); ++b; }
    }
  }
  size_t take = size_t(2 * m - 2);
  for (int d = 1; d <= maxlen && take; ++d) {
    size_t npk = 0;
    for (size_t i = 0; i < take && i < lists[d].size(); ++i) {
      if (lists[d][i].sym >= 0) ++lens[lists[d][i].sym];
      else ++npk;
    }
    take = 2 * npk;
  }
}

// canonical codes (RFC 1951 §3.2.2), returned bit-reversed for LSB-first emission
void canonical_rev(const uint8_t* lens, int n, uint32_t* rev) {
  uint32_t count[16] = {0}, next[16] = {0};
  for (int i = 0; i < n; ++i) ++count[lens[i]];
  count[0] = 0;
  uint32_t code = 0;
  for (int b = 1; b <= 15; ++b) { code = (code + count[b - 1]) << 1; next[b] = code; }
  for (int i = 0; i < n; ++i) {
    rev[i] = 0;
    if (!lens[i]) continue;
    uint32_t c = next[lens[i]]++, r = 0;
    for (int k = 0; k < lens[i]; ++k) r |= ((c >> k) & 1u) << (lens[i] - 1 - k);
    rev[i] = r;
  }
}

struct BitWriter {
  std::vector<uint8_t>& out;
  uint64_t acc = 0;
  int n = 0;
  uint64_t total = 0;
  explicit BitWriter(std::vector<uint8_t>& o) : out(o) {}
  void put(uint32_t v, int bits) {  // LSB-first
    acc |= uint64_t(v) << n;
    n += bits;
    total += uint64_t(bits);
    while (n >= 8) { out.push_back(uint8_t(acc)); acc >>= 8; n -= 8; }
  }
  void flush() { if (n > 0) { out.push_back(uint8_t(acc)); acc = 0; n = 0; } }
};

struct BlockOut {
  std::vector<uint8_t> payload;
  uint32_t n_seq = 0, n_lit = 0, S = 0, n_sub = 0;
  std::vector<uint32_t> sub;  // (bit_size, n_lit) pairs
  gomp_status st = GOMP_OK;
};

void encode_block(const uint8_t* blk, uint32_t n, const gomp_params& p, const std::vector<Seq>& seqs, BlockOut& o) {
  o.n_seq = uint32_t(seqs.size());
  o.n_lit = 0;
  for (const Seq& q : seqs) o.n_lit += q.lit;
  o.payload.clear();
  if (p.mode == GOMP_MODE_BYTE) {
    o.payload.resize(align16(4ull * o.n_seq + o.n_lit), 0);
    uint8_t* lits = o.payload.data() + 4ull * o.n_seq;
    uint32_t c = 0, lp = 0;
    for (uint32_t i = 0; i < o.n_seq; ++i) {
      const Seq& q = seqs[i];
      const uint32_t mcode = q.L ? q.L - p.min_match + 1 : 0;
      st32(o.payload.data() + 4ull * i, q.lit | mcode << 10 | (q.L ? (q.dist - 1) << 16 : 0u));
      std::memcpy(lits + lp, blk + c, q.lit);
      lp += q.lit;
      c += q.lit + q.L;
    }
    return;
  }
  uint64_t fl[286] = {0}, fd[30] = {0};
  uint32_t c = 0;
  for (const Seq& q : seqs) {
    for (uint32_t k = 0; k < q.lit; ++k) ++fl[blk[c + k]];
    if (q.L) { ++fl[257 + len_index(q.L)]; ++fd[dist_index(q.dist)]; }
    c += q.lit + q.L;
  }
  ++fl[256];
  uint8_t ll[286], dl[30];
  uint32_t lr[286], dr[30];
  package_merge(fl, 286, int(p.cwl), ll);
  package_merge(fd, 30, int(p.cwl), dl);
  bool any = false;
  for (int i = 0; i < 30; ++i) any |= dl[i] != 0;
  if (!any) dl[0] = 1;  // R14: one dummy distance code
  canonical_rev(ll, 286, lr);
  canonical_rev(dl, 30, dr);
  o.payload.assign(kTreeBytes, 0);
  for (int i = 0; i < 286; ++i) o.payload[i / 2] |= uint8_t(ll[i] << (4 * (i & 1)));
  for (int i = 0; i < 30; ++i) o.payload[143 + i / 2] |= uint8_t(dl[i] << (4 * (i & 1)));
  o.S = p.sub_block_seqs ? p.sub_block_seqs : (o.n_seq + p.sub_blocks_per_block - 1) / p.sub_blocks_per_block;
  if (o.S == 0) o.S = 1;
  o.n_sub = (o.n_seq + o.S - 1) / o.S;
  o.sub.assign(2ull * o.n_sub, 0);
  o.payload.reserve(kTreeBytes + n + n / 2 + 64);
  BitWriter w(o.payload);
  c = 0;
  uint32_t k = 0;
  for (uint32_t sb = 0; sb < o.n_sub; ++sb) {
    const uint64_t bit0 = w.total;
    uint32_t nl = 0;
    const uint32_t end = std::min<uint64_t>(uint64_t(sb + 1) * o.S, o.n_seq);
    for (; k < end; ++k) {
      const Seq& q = seqs[k];
      for (uint32_t t = 0; t < q.lit; ++t) { const uint8_t b = blk[c + t]; w.put(lr[b], ll[b]); }
      nl += q.lit;
      if (q.L) {
        const int li = len_index(q.L), di = dist_index(q.dist);
        w.put(lr[257 + li], ll[257 + li]);
        w.put(q.L - kLenBase[li], kLenExtra[li]);
        w.put(dr[di], dl[di]);
        w.put(q.dist - kDistBase[di], kDistExtra[di]);
      }
      c += q.lit + q.L;
    }
    if (sb + 1 == o.n_sub) w.put(lr[256], ll[256]);  // EOB closes the block
    o.sub[2 * sb] = uint32_t(w.total - bit0);
    o.sub[2 * sb + 1] = nl;
  }
  w.flush();
  o.payload.resize(align16(o.payload.size()), 0);
  (void)n;
}

bool params_ok(const gomp_params* p) {
  if (!p || p->struct_size != sizeof(gomp_params)) return false;
  if (p->mode > 1 || p->block_size < 16 || p->block_size % 16 || p->window_size < 1 || p->window_size > 32768) return false;
  if ((p->min_match != 3 && p->min_match != 4) || p->max_match < p->min_match || p->max_match > p->min_match + 62) return false;
  if (p->match_finder > 1) return false;
  if (p->de_group == 0 || p->de_group % kGroup || p->de_group > 224) return false;
  if (p->mode == GOMP_MODE_BIT) {
    if (p->cwl < 9 || p->cwl > 15) return false;
    if (p->sub_block_seqs == 0 && p->sub_blocks_per_block == 0) return false;
  }
  return true;
}

uint64_t max_seqs(uint32_t bs, uint32_t mm) { return uint64_t(bs) / mm + bs / kMaxLitRun + 2; }

uint64_t block_bound(const gomp_params* p) {
  const uint64_t bs = p->block_size, ns = max_seqs(p->block_size, p->min_match);
  if (p->mode == GOMP_MODE_BYTE) return kBlockEntryBytes + align16(4 * ns + bs) + 16;
  const uint64_t S = p->sub_block_seqs ? p->sub_block_seqs : 1;
  const uint64_t nsub = p->sub_block_seqs ? ns / S + 1 : p->sub_blocks_per_block;
  return kBlockEntryBytes + kSubEntryBytes * nsub + kTreeBytes + (15 * bs + 48 * ns) / 8 + 64;
}

}  // namespace

// internal interface for the GPU compressor (compress_gpu.cu): the same parameter checks, package-merge and
// header layout as the host compressor, so both produce identical files
bool host_params_ok(const gomp_params* p) { return params_ok(p); }
uint64_t host_max_seqs(uint32_t bs, uint32_t mm) { return max_seqs(bs, mm); }
void host_write_header(uint8_t* h, const gomp_params* p, uint32_t nb, uint64_t src_len, uint64_t file_len,
                       uint64_t n_sub_total, uint64_t max_tok, uint64_t base) {
  std::memcpy(h, "GMPR", 4);
  h[4] = 1;
  h[5] = uint8_t(p->mode);
  h[6] = p->de ? 1 : 0;
  h[7] = uint8_t(p->min_match);
  h[8] = uint8_t(p->max_match);
  h[9] = uint8_t(p->mode == GOMP_MODE_BIT ? p->cwl : 0);
  h[10] = uint8_t(p->de_group);
  h[11] = 0;
  st32(h + 12, p->block_size);
  st32(h + 16, p->window_size);
  st32(h + 20, nb);
  st64(h + 24, src_len);
  st64(h + 32, file_len);
  st32(h + 40, uint32_t(n_sub_total));
  st32(h + 44, p->mode == GOMP_MODE_BIT ? uint32_t(max_tok) : 0);
  st64(h + 48, base);
  st32(h + 56, 0);
  st32(h + 60, 0);
}
}  // namespace gomp

using namespace gomp;

extern "C" {

__attribute__((visibility("default"))) void gomp_params_default(gomp_params* p) {
  if (!p) return;
  std::memset(p, 0, sizeof(*p));
  p->struct_size = sizeof(gomp_params);
  p->mode = GOMP_MODE_BIT;
  p->de = 1;
  p->block_size = 262144;   // 256 KB blocks
  p->window_size = 8192;    // 8 KB window
  p->min_match = 4;         // R8
  p->max_match = 64;        // 64-byte lookahead
  p->sub_block_seqs = 16;   // 16-sequence sub-blocks
  p->sub_blocks_per_block = 0;
  p->cwl = 10;              // CWL = 10 bits
  p->match_finder = 0;
  p->min_staleness = 1024;
  p->max_chain = 0;
  p->n_threads = 0;
  p->de_group = kGroup;     // 32-sequence warp groups
}

__attribute__((visibility("default"))) size_t gomp_compress_bound(size_t src_len, const gomp_params* p) {
  if (!params_ok(p)) return 0;
  const uint64_t nb = (src_len + p->block_size - 1) / p->block_size;
  return size_t(kHeaderBytes + nb * block_bound(p) + 16 + kTrailerBytes);
}

__attribute__((visibility("default"))) gomp_status gomp_compress(const uint8_t* src, size_t src_len, uint8_t* dst,
                                                                 size_t dst_cap, size_t* dst_len, const gomp_params* p) {
  if (!params_ok(p) || !dst || !dst_len || (!src && src_len)) return GOMP_ERR_INVALID_ARG;
  const uint64_t nb64 = (uint64_t(src_len) + p->block_size - 1) / p->block_size;
  if (nb64 > 0xffffffffull) return GOMP_ERR_INVALID_ARG;
  const uint32_t nb = uint32_t(nb64);
  std::vector<BlockOut> blocks;
  try {
    blocks.resize(nb);
  } catch (const std::bad_alloc&) {
    return GOMP_ERR_OOM;
  }
  unsigned nt = p->n_threads ? p->n_threads : std::max(1u, std::thread::hardware_concurrency());
  nt = std::min<unsigned>(nt, std::max<uint32_t>(nb, 1));
  std::atomic<uint32_t> next{0};
  std::atomic<int> oom{0};
  auto worker = [&]() {
    ParseScratch scratch;
    std::vector<Seq> seqs;
    try {
      for (;;) {
        const uint32_t b = next.fetch_add(1);
        if (b >= nb) break;
        const uint64_t off = uint64_t(b) * p->block_size;
        const uint32_t n = uint32_t(std::min<uint64_t>(p->block_size, src_len - off));
        seqs.clear();
        parse_block(src + off, n, *p, seqs, scratch);
        encode_block(src + off, n, *p, seqs, blocks[b]);
      }
    } catch (const std::bad_alloc&) {
      oom = 1;
    }
  };
  if (nt <= 1) {
    worker();
  } else {
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t) th.emplace_back(worker);
    for (auto& t : th) t.join();
  }
  if (oom) return GOMP_ERR_OOM;
  uint64_t n_sub_total = 0, max_tok = 0;
  for (const BlockOut& o : blocks) {
    n_sub_total += o.n_sub;
    max_tok = std::max<uint64_t>(max_tok, 4ull * o.n_seq + o.n_lit);
  }
  if (n_sub_total > 0xffffffffull) return GOMP_ERR_INVALID_ARG;
  const uint64_t base = align16(kHeaderBytes + uint64_t(kBlockEntryBytes) * nb + uint64_t(kSubEntryBytes) * n_sub_total);
  uint64_t total = base;
  for (const BlockOut& o : blocks) total += o.payload.size();
  total += kTrailerBytes;
  if (total > dst_cap) return GOMP_ERR_DST_TOO_SMALL;
  std::memset(dst, 0, base);
  uint64_t pos = base;
  uint32_t sub_at = 0;
  for (uint32_t b = 0; b < nb; ++b) {
    const BlockOut& o = blocks[b];
    uint8_t* e = dst + kHeaderBytes + uint64_t(kBlockEntryBytes) * b;
    st64(e, pos);
    st32(e + 8, uint32_t(o.payload.size()));
    st32(e + 12, o.n_seq);
    st32(e + 16, o.n_lit);
    st32(e + 20, p->mode == GOMP_MODE_BIT ? sub_at : 0);
    st32(e + 24, o.S);
    st32(e + 28, o.n_sub);
    for (uint32_t k = 0; k < o.n_sub; ++k) {
      uint8_t* s = dst + kHeaderBytes + uint64_t(kBlockEntryBytes) * nb + uint64_t(kSubEntryBytes) * (sub_at + k);
      st32(s, o.sub[2 * k]);
      st32(s + 4, o.sub[2 * k + 1]);
    }
    sub_at += o.n_sub;
    std::memcpy(dst + pos, o.payload.data(), o.payload.size());
    pos += o.payload.size();
  }
  std::memset(dst + pos, 0, kTrailerBytes);
  pos += kTrailerBytes;
  host_write_header(dst, p, nb, src_len, pos, n_sub_total, max_tok, base);
  *dst_len = size_t(pos);
  return GOMP_OK;
}

}  // extern "C"
