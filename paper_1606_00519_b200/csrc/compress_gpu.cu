// compress_gpu.cu — Gompresso compression on the GPU: the producer of the
// decoder's input, writing the same file as the host compressor gomp_compress (match_finder 0) byte for byte.
//
//   lz_parse_kernel     one warp per data block ("each block is LZ77-compressed by a group of threads"):
//                       the greedy longest-match parse of FORMAT.md §2 with Dependency Elimination (Fig.
//                       alg:dedeflate P:256-284; readings R2/R4/R5/R7/R10/R22). Candidates = every earlier
//                       position of the window whose first min_match bytes hash like the cursor's (hash chains
//                       in shared memory, inserted 32 positions per warp step with __match_any_sync); a match of
//                       length >= min_match shares those bytes, so the candidate set, its nearest-first order
//                       and hence the parse equal the exhaustive search. Lane 0 walks up to 32 chain links, the
//                       32 lanes compare them in parallel (word compares), a warp max-reduction picks the longest
//                       (ties: smallest distance). Output: Byte-format records per block.
//   byte_payload_kernel Gompresso/Byte payloads: records + the literal strings gathered from the input.
//   freq_kernel         Gompresso/Bit: per-block literal/length and distance symbol counts (RFC 1951 alphabet, R15).
//   pm_kernel           package-merge code lengths <= CWL per block (R14; the host compressor's algorithm and tie
//                       order, so the files stay identical) and the sub-block size S (R12), on the device.
//   huff_encode_kernel  canonical codes, per-sequence bit counts, a block-wide scan of bit offsets,
//                       then every thread writes its sequence's bits (LSB-first, R15) at its offset: interior
//                       32-bit words by plain stores, the two boundary words by atomicOr; sub-block bit sizes
//                       and literal counts for the sub-block table (R12/R13).
//   place_kernel        payloads to their final, 16-byte aligned file offsets.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

#include "compress.hpp"
#include "format.hpp"
#include "gomp.h"

#define GOMP_EXPORT extern "C" __attribute__((visibility("default")))

namespace gomp {
namespace {

constexpr uint32_t FULLM = 0xffffffffu;
constexpr uint32_t kHashBits = 11;                 // chain buckets (collisions are filtered by the compare)
constexpr uint32_t kParseWarps = 4;                // warps (= data blocks) per CTA of the parse kernel
constexpr uint32_t kCompThreads = 512;             // threads per CTA of the per-block encode kernels
constexpr uint32_t kNoPos = 0xffffffffu;

__constant__ uint16_t k_len_base[29] = {3,  4,  5,  6,  7,  8,  9,  10, 11,  13,  15,  17,  19,  23, 27,
                                        31, 35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
__constant__ uint8_t k_len_extra[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
__constant__ uint16_t k_dist_base[30] = {1,    2,    3,    4,    5,    7,    9,    13,    17,    25,
                                         33,   49,   65,   97,   129,  193,  257,  385,   513,   769,
                                         1025, 1537, 2049, 3073, 4097, 6145, 8193, 12289, 16385, 24577};
__constant__ uint8_t k_dist_extra[30] = {0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};

__device__ __forceinline__ uint32_t len_code(uint32_t L) {   // RFC 1951 §3.2.5 length code index
  if (L == 258) return 28;
  uint32_t i = 27;
  while (k_len_base[i] > L) --i;
  return i;
}
__device__ __forceinline__ uint32_t dist_code(uint32_t d) {
  uint32_t i = 29;
  while (k_dist_base[i] > d) --i;
  return i;
}

struct CArgs {
  const uint8_t* src;     // the input, copied into the workspace with >= 16 zero bytes behind it
  uint64_t src_len;
  uint32_t nb, block_size, window, mm, maxm, de, de_group, max_seqs, pm;   // pm: prev-ring mask
  uint32_t* recs;         // block b: recs + b * max_seqs (Byte-format records, FORMAT.md §3)
  uint32_t* meta;         // block b: {n_seq, n_lit, bits (Bit), payload bytes}
};

__device__ __forceinline__ uint32_t word_at(const uint8_t* blk, uint32_t x) {   // bytes x..x+3, little-endian
  const uint32_t* p = reinterpret_cast<const uint32_t*>(reinterpret_cast<uintptr_t>(blk + x) & ~uintptr_t(3));
  return __funnelshift_r(__ldg(p), __ldg(p + 1), (uint32_t(reinterpret_cast<uintptr_t>(blk + x)) & 3u) * 8u);
}
__device__ __forceinline__ uint32_t hash_mm(uint32_t w, uint32_t mm) {
  const uint32_t v = mm == 4 ? w : (w & 0xffffffu);
  return (v * 2654435761u) >> (32 - kHashBits);
}

// ------------------------------------------------------------------ LZ77 parse, one warp per block
__global__ void __launch_bounds__(32 * kParseWarps) lz_parse_kernel(const CArgs a) {
  extern __shared__ __align__(16) uint8_t psm[];
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t b = blockIdx.x * nw + w;
  if (b >= a.nb) return;
  const uint32_t PR = a.pm + 1;
  // per warp: head[2^kHashBits] | cand[32] (u32), then the prev rings of all warps (u16 distance to the previous
  // position of the same bucket, 0 = none within the window)
  uint32_t* head = reinterpret_cast<uint32_t*>(psm) + w * ((1u << kHashBits) + 32);
  uint32_t* cand = head + (1u << kHashBits);
  uint16_t* prev = reinterpret_cast<uint16_t*>(reinterpret_cast<uint32_t*>(psm) + nw * ((1u << kHashBits) + 32)) +
                   w * PR;
  for (uint32_t i = lane; i < (1u << kHashBits); i += 32) head[i] = kNoPos;
  __syncwarp();
  const uint64_t off = uint64_t(b) * a.block_size;
  const uint64_t rem = a.src_len - off;
  const uint32_t n = rem < a.block_size ? uint32_t(rem) : a.block_size;
  const uint8_t* blk = a.src + off;
  uint32_t* rec = a.recs + uint64_t(b) * a.max_seqs;
  const uint32_t mm = a.mm, win = a.window, G = a.de_group;
  uint32_t c = 0, ls = 0, nseq = 0, hwm = 0, ins = 0, nlit = 0;
  auto emit = [&](uint32_t lit, uint32_t L, uint32_t d) {
    if (lane == 0) rec[nseq] = lit | (L ? ((L - mm + 1) << 10) | ((d - 1) << 16) : 0u);
    nlit += lit;
    if (++nseq % G == 0) hwm = c;   // warpHWM <- pos after every de_group sequences (R22)
  };
  const uint32_t ins_end = n >= mm ? n - mm + 1 : 0;   // positions that can start a min_match-byte match
  while (c < n) {
    // index every position < c (nearest-first chains; a batch of 32 positions per step)
    const uint32_t iend = min(c, ins_end);
    while (ins < iend) {
      const uint32_t p = ins + lane;
      const bool v = p < iend;
      const uint32_t h = v ? hash_mm(word_at(blk, p), mm) : (0x80000000u | lane);
      const uint32_t same = __match_any_sync(FULLM, h);
      const uint32_t lower = same & ((1u << lane) - 1u);
      const uint32_t older = lower ? ins + (31 - __clz(lower)) : (v ? head[h] : kNoPos);
      __syncwarp();
      if (v) {
        const uint32_t d = older == kNoPos ? 0u : p - older;
        prev[p & a.pm] = uint16_t(d <= win ? d : 0u);        // 0: end of chain (or beyond the window)
        if ((same >> lane) == 1u) head[h] = p;                 // highest lane of its bucket
      }
      __syncwarp();
      ins = min(ins + 32, iend);
    }
    if (ins < c) ins = c;   // positions too close to the block end to start a match are never indexed
    uint32_t best = 0, bdist = 0;
    const uint32_t maxL = min(a.maxm, n - c);
    if (maxL >= mm) {
      const uint32_t P = word_at(blk, c);
      uint32_t s = head[hash_mm(P, mm)];
      uint32_t key = 0;   // (len << 16) | (0xffff - dist): max = longest, then nearest
      while (s != kNoPos && c - s <= win) {
        // lane 0 walks up to 32 links of the chain, then the warp compares them in parallel
        uint32_t nc = 0;
        if (lane == 0) {
          uint32_t t = s;
          while (nc < 32 && t != kNoPos && c - t <= win) {
            cand[nc++] = t;
            const uint32_t d = prev[t & a.pm];
            t = d ? t - d : kNoPos;
          }
          s = t;
        }
        __syncwarp();
        nc = __shfl_sync(FULLM, nc, 0);
        s = __shfl_sync(FULLM, s, 0);
        uint32_t lk = 0;
        if (lane < nc) {
          const uint32_t sp = cand[lane];
          uint32_t cap = min(maxL, c - sp);   // no overlap (R2)
          bool ok = true;
          if (a.de && sp < ls) {              // DE (R4/R5): below warpHWM, truncated to it
            if (sp >= hwm) ok = false;
            else cap = min(cap, hwm - sp);
          }
          if (ok && cap >= mm && cap > (key >> 16)) {
            uint32_t len = 0;
            for (;;) {
              const uint32_t x = word_at(blk, sp + len) ^ word_at(blk, c + len);
              if (x) { len += (__ffs(x) - 1) >> 3; break; }
              len += 4;
              if (len >= cap) break;
            }
            len = min(len, cap);
            if (len >= mm) lk = (len << 16) | (0xffffu - (c - sp));
          }
        }
        key = max(key, __reduce_max_sync(FULLM, lk));
        __syncwarp();
        if ((key >> 16) >= maxL) break;
      }
      best = key >> 16;
      bdist = 0xffffu - (key & 0xffffu);
    }
    if (best >= mm) {
      const uint32_t lit = c - ls;
      c += best;
      emit(lit, best, bdist);
      ls = c;
    } else {
      ++c;
      if (c - ls == kMaxLitRun) {   // R10: close a literal run at 1023 bytes
        emit(kMaxLitRun, 0, 0);
        ls = c;
      }
    }
  }
  if (c > ls) emit(c - ls, 0, 0);
  if (lane == 0) {
    a.meta[4 * b] = nseq;
    a.meta[4 * b + 1] = nlit;
  }
}

// CTA-wide exclusive scan of one value per thread (blockDim.x = kCompThreads); returns the exclusive prefix
// and the total through *tot
__device__ __forceinline__ uint32_t cta_scan(uint32_t v, uint32_t* wsum, uint32_t* tot) {
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_up_sync(FULLM, x, d);
    if (lane >= uint32_t(d)) x += t;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t y = lane < kCompThreads / 32 ? wsum[lane] : 0u;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(FULLM, y, d);
      if (lane >= uint32_t(d)) y += t;
    }
    if (lane < kCompThreads / 32) wsum[lane] = y;
  }
  __syncthreads();
  const uint32_t pre = (w ? wsum[w - 1] : 0u) + x - v;
  *tot = wsum[kCompThreads / 32 - 1];
  __syncthreads();
  return pre;
}

// ------------------------------------------------------------------ Byte payloads (records + literals)
__global__ void __launch_bounds__(kCompThreads) byte_payload_kernel(const CArgs a, uint8_t* dst, const uint64_t* pos) {
  __shared__ uint32_t wsum[kCompThreads / 32];
  const uint32_t b = blockIdx.x, ns = a.meta[4 * b];
  const uint32_t* rec = a.recs + uint64_t(b) * a.max_seqs;
  const uint8_t* blk = a.src + uint64_t(b) * a.block_size;
  uint8_t* out = dst + pos[b];
  uint8_t* lits = out + 4ull * ns;
  const uint32_t nlit = a.meta[4 * b + 1], plen = (4 * ns + nlit + 15u) & ~15u;
  uint32_t ocar = 0, lcar = 0;
  for (uint32_t i0 = 0; i0 < ns; i0 += kCompThreads) {
    const uint32_t i = i0 + threadIdx.x;
    const uint32_t r = i < ns ? rec[i] : 0u;
    const uint32_t lit = r & 1023u, mc = (r >> 10) & 63u, L = mc ? mc + a.mm - 1 : 0u;
    uint32_t t1, t2;
    const uint32_t op = ocar + cta_scan(lit + L, wsum, &t1);
    const uint32_t lp = lcar + cta_scan(lit, wsum, &t2);
    if (i < ns) {
      reinterpret_cast<uint32_t*>(out)[i] = r;
      for (uint32_t k = 0; k < lit; ++k) lits[lp + k] = blk[op + k];
    }
    ocar += t1;
    lcar += t2;
  }
  for (uint32_t p = 4 * ns + nlit + threadIdx.x; p < plen; p += kCompThreads) out[p] = 0;
}

// ------------------------------------------------------------------ Bit: symbol counts per block
__global__ void __launch_bounds__(kCompThreads) freq_kernel(const CArgs a, uint32_t* freq) {
  __shared__ uint32_t wsum[kCompThreads / 32];
  __shared__ uint32_t fl[316];
  const uint32_t b = blockIdx.x, ns = a.meta[4 * b];
  for (uint32_t s = threadIdx.x; s < 316; s += kCompThreads) fl[s] = 0;
  __syncthreads();
  const uint32_t* rec = a.recs + uint64_t(b) * a.max_seqs;
  const uint8_t* blk = a.src + uint64_t(b) * a.block_size;
  uint32_t ocar = 0;
  for (uint32_t i0 = 0; i0 < ns; i0 += kCompThreads) {
    const uint32_t i = i0 + threadIdx.x;
    const uint32_t r = i < ns ? rec[i] : 0u;
    const uint32_t lit = r & 1023u, mc = (r >> 10) & 63u, L = mc ? mc + a.mm - 1 : 0u, d = (r >> 16) + 1u;
    uint32_t t;
    const uint32_t op = ocar + cta_scan(lit + L, wsum, &t);
    if (i < ns) {
      for (uint32_t k = 0; k < lit; ++k) atomicAdd(&fl[blk[op + k]], 1u);
      if (L) {
        atomicAdd(&fl[257 + len_code(L)], 1u);
        atomicAdd(&fl[286 + dist_code(d)], 1u);
      }
    }
    ocar += t;
  }
  __syncthreads();
  if (threadIdx.x == 0) fl[256] += 1;   // EOB
  __syncthreads();
  for (uint32_t s = threadIdx.x; s < 316; s += kCompThreads) freq[316ull * b + s] = fl[s];
}

// Package-merge code lengths <= cwl (R14) on the device, per block: warp 0 the 286 literal/length symbols, warp 1
// the 30 distance symbols. The same algorithm and tie order as the host routine (compress.cpp package_merge):
// leaves are the used symbols ordered by (frequency, symbol) (a warp rank sort), lists[cwl] = the leaves,
// lists[d] = merge(leaves, pairs of lists[d+1]) with a leaf before a package of equal weight; the first 2m - 2
// items of lists[1] are selected, a selected package selects the first 2P items of the next list, and a symbol's
// length is the number of times it is selected. Lane 0 runs the merge (at most 2m - 1 items per list, 15 lists);
// lane 0 of warp 2 derives the block's sub-block size S (R12). No host round trip between freq and encode.
template <uint32_t N>   // alphabet size; a list holds at most 2N - 1 items
struct PmSmem {
  uint64_t w[2][2 * N];                // item weights of the previous and the current list
  int16_t item[16][2 * N];             // item kinds per list: symbol (leaf) or -1 (package)
  uint16_t cnt[16];                    // items per list
  uint16_t sorted[N];
  uint32_t f[N];
};
template <uint32_t N>
__device__ void pm_table(PmSmem<N>& sm, const uint32_t* fr, uint32_t n, uint32_t maxlen, uint8_t* lens, uint32_t lane) {
  // used symbols ranked by (frequency, symbol)
  for (uint32_t i = lane; i < n; i += 32) sm.f[i] = fr[i];
  __syncwarp();
  uint32_t m = 0;
  for (uint32_t i = lane; i < n; i += 32) {
    const uint32_t fi = sm.f[i];
    if (fi) {
      uint32_t r = 0;
      for (uint32_t j = 0; j < n; ++j) {
        const uint32_t fj = sm.f[j];
        r += fj && (fj < fi || (fj == fi && j < i));
      }
      sm.sorted[r] = uint16_t(i);
    }
    m += fi != 0;
  }
  for (int d = 16; d; d >>= 1) m += __shfl_xor_sync(FULLM, m, d);
  for (uint32_t i = lane; i < n; i += 32) lens[i] = 0;
  __syncwarp();
  if (lane != 0 || m == 0) return;
  if (m == 1) { lens[sm.sorted[0]] = 1; return; }
  uint32_t cur = 0;
  for (uint32_t i = 0; i < m; ++i) {
    sm.w[cur][i] = sm.f[sm.sorted[i]];
    sm.item[maxlen][i] = int16_t(sm.sorted[i]);
  }
  sm.cnt[maxlen] = uint16_t(m);
  for (uint32_t d = maxlen - 1; d >= 1; --d) {
    const uint32_t np = sm.cnt[d + 1] / 2, nx = cur ^ 1u;
    uint32_t a = 0, b = 0, k = 0;
    while (a < m || b < np) {
      const uint64_t pw = b < np ? sm.w[cur][2 * b] + sm.w[cur][2 * b + 1] : 0ull;
      const uint64_t lw = a < m ? uint64_t(sm.f[sm.sorted[a]]) : 0ull;
      if (b >= np || (a < m && lw <= pw)) {
        sm.w[nx][k] = lw;
        sm.item[d][k] = int16_t(sm.sorted[a]);
        ++a;
      } else {
        sm.w[nx][k] = pw;
        sm.item[d][k] = -1;
        ++b;
      }
      ++k;
    }
    sm.cnt[d] = uint16_t(k);
    cur = nx;
  }
  uint32_t take = 2 * m - 2;
  for (uint32_t d = 1; d <= maxlen && take; ++d) {
    uint32_t npk = 0;
    for (uint32_t i = 0; i < take && i < sm.cnt[d]; ++i) {
      const int s = sm.item[d][i];
      if (s >= 0) ++lens[s];
      else ++npk;
    }
    take = 2 * npk;
  }
}

__global__ void __launch_bounds__(96) pm_kernel(const CArgs a, const uint32_t* freq, uint8_t* lens_out, uint32_t* Sb,
                                                uint32_t cwl, uint32_t sub_block_seqs, uint32_t sub_blocks_per_block) {
  __shared__ PmSmem<286> sml;
  __shared__ PmSmem<30> smd;
  __shared__ uint8_t lens[316];
  const uint32_t b = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t* fr = freq + 316ull * b;
  if (w == 0) pm_table(sml, fr, 286, cwl, lens, lane);
  else if (w == 1) pm_table(smd, fr + 286, 30, cwl, lens + 286, lane);
  else if (lane == 0) {
    const uint32_t ns = a.meta[4 * b];
    uint32_t S = sub_block_seqs ? sub_block_seqs : (ns + sub_blocks_per_block - 1) / sub_blocks_per_block;
    Sb[b] = S ? S : 1u;
  }
  __syncthreads();
  if (threadIdx.x == 0) {   // R14: a block without back-references gets one dummy distance code
    bool any = false;
    for (int i = 0; i < 30; ++i) any |= lens[286 + i] != 0;
    if (!any) lens[286] = 1;
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < 316; i += blockDim.x) lens_out[316ull * b + i] = lens[i];
}

// ------------------------------------------------------------------ Bit: encode one block
// Writes the bits of one sequence, range [b0, b1) of the block stream, LSB-first: pending bits accumulate in a
// 64-bit register; a 32-bit word is emitted once its last bit is pending: a plain store when the word lies wholly
// inside [b0, b1), an atomicOr when a neighbouring sequence owns some of its bits (the stream is zeroed first).
struct SeqWriter {
  uint32_t* words;
  uint64_t b0, b1, at;   // at: next bit position
  uint64_t acc;          // nacc pending bits, the first at position at - nacc
  uint32_t nacc;
  __device__ __forceinline__ void put(uint32_t v, uint32_t bits) {
    acc |= uint64_t(v) << nacc;
    nacc += bits;
    at += bits;
    for (;;) {
      const uint64_t start = at - nacc;
      const uint32_t sh = uint32_t(start & 31), take = 32 - sh;
      if (nacc < take) break;
      const uint64_t wi = start >> 5;
      const uint32_t v32 = uint32_t(acc << sh);
      if (sh == 0 && (wi << 5) >= b0 && (wi << 5) + 32 <= b1) words[wi] = v32;
      else atomicOr(&words[wi], v32);
      acc >>= take;
      nacc -= take;
    }
  }
  __device__ __forceinline__ void finish() {   // the last partial word (fewer than 32 - (start & 31) bits)
    if (nacc) {
      const uint64_t start = at - nacc;
      atomicOr(&words[start >> 5], uint32_t(acc << (start & 31)));
    }
  }
};

__global__ void __launch_bounds__(kCompThreads) huff_encode_kernel(const CArgs a, const uint8_t* lens, uint8_t* pay,
                                                                   uint64_t pay_stride, uint32_t* subtab,
                                                                   uint32_t sub_stride, const uint32_t* Sb) {
  __shared__ uint32_t wsum[kCompThreads / 32];
  __shared__ uint32_t code[316];
  __shared__ uint8_t clen[316];
  __shared__ uint32_t subbits[1024], sublits[1024];
  const uint32_t b = blockIdx.x, ns = a.meta[4 * b];
  const uint8_t* L8 = lens + 316ull * b;
  uint8_t* out = pay + uint64_t(b) * pay_stride;
  // canonical codes (RFC 1951 §3.2.2), bit-reversed for LSB-first emission; the tree nibbles (R18)
  if (threadIdx.x < 2) {
    const uint32_t t = threadIdx.x, n = t ? 30u : 286u, o = t ? 286u : 0u;
    uint32_t count[16] = {0}, next[16] = {0};
    for (uint32_t i = 0; i < n; ++i) ++count[L8[o + i]];
    count[0] = 0;
    uint32_t cd = 0;
    for (int k = 1; k <= 15; ++k) { cd = (cd + count[k - 1]) << 1; next[k] = cd; }
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t l = L8[o + i];
      clen[o + i] = uint8_t(l);
      code[o + i] = l ? __brev(next[l]++) >> (32 - l) : 0u;
    }
  }
  for (uint32_t i = threadIdx.x; i < kTreeBytes; i += kCompThreads) {
    uint32_t v = 0;
    if (i < 143) v = L8[2 * i] | (2 * i + 1 < 286 ? uint32_t(L8[2 * i + 1]) << 4 : 0u);
    else if (i < 158) v = L8[286 + 2 * (i - 143)] | (uint32_t(L8[286 + 2 * (i - 143) + 1]) << 4);
    out[i] = uint8_t(v);
  }
  const uint32_t S = Sb[b], nsub = ns ? (ns + S - 1) / S : 0;
  for (uint32_t k = threadIdx.x; k < nsub && k < 1024; k += kCompThreads) { subbits[k] = 0; sublits[k] = 0; }
  __syncthreads();
  uint32_t* words = reinterpret_cast<uint32_t*>(out + kTreeBytes);
  const uint8_t* blk = a.src + uint64_t(b) * a.block_size;
  const uint32_t* rec = a.recs + uint64_t(b) * a.max_seqs;
  uint32_t ocar = 0, bcar = 0;
  for (uint32_t i0 = 0; i0 < ns; i0 += kCompThreads) {
    const uint32_t i = i0 + threadIdx.x;
    const uint32_t r = i < ns ? rec[i] : 0u;
    const uint32_t lit = r & 1023u, mc = (r >> 10) & 63u, L = mc ? mc + a.mm - 1 : 0u, d = (r >> 16) + 1u;
    uint32_t t1, t2;
    const uint32_t op = ocar + cta_scan(lit + L, wsum, &t1);
    // this sequence's bits: literal codes, then length code + extra, distance code + extra; the block's last
    // sequence is followed by EOB (it closes the last sub-block, FORMAT.md §3)
    uint32_t nb = 0, li = 0, di = 0;
    if (i < ns) {
      for (uint32_t k = 0; k < lit; ++k) nb += clen[blk[op + k]];
      if (L) {
        li = len_code(L);
        di = dist_code(d);
        nb += clen[257 + li] + k_len_extra[li] + clen[286 + di] + k_dist_extra[di];
      }
      if (i + 1 == ns) nb += clen[256];
    }
    const uint32_t bit0 = bcar + cta_scan(nb, wsum, &t2);
    if (i < ns) {
      SeqWriter wr{words, bit0, uint64_t(bit0) + nb, bit0, 0ull, 0u};
      for (uint32_t k = 0; k < lit; ++k) { const uint32_t y = blk[op + k]; wr.put(code[y], clen[y]); }
      if (L) {
        wr.put(code[257 + li], clen[257 + li]);
        wr.put(L - k_len_base[li], k_len_extra[li]);
        wr.put(code[286 + di], clen[286 + di]);
        wr.put(d - k_dist_base[di], k_dist_extra[di]);
      }
      if (i + 1 == ns) wr.put(code[256], clen[256]);
      wr.finish();
      const uint32_t k = i / S;
      if (k < 1024) {
        atomicAdd(&subbits[k], nb);
        atomicAdd(&sublits[k], lit);
      } else {
        atomicAdd(&subtab[uint64_t(b) * sub_stride + 2 * k], nb);
        atomicAdd(&subtab[uint64_t(b) * sub_stride + 2 * k + 1], lit);
      }
    }
    ocar += t1;
    bcar += t2;
  }
  __syncthreads();
  for (uint32_t k = threadIdx.x; k < nsub && k < 1024; k += kCompThreads) {
    subtab[uint64_t(b) * sub_stride + 2 * k] = subbits[k];
    subtab[uint64_t(b) * sub_stride + 2 * k + 1] = sublits[k];
  }
  if (threadIdx.x == 0) a.meta[4 * b + 2] = bcar;
}

__global__ void place_kernel(const uint8_t* pay, uint64_t pay_stride, const uint32_t* meta, const uint64_t* pos,
                             uint8_t* dst) {
  const uint32_t b = blockIdx.x, len = meta[4 * b + 3];
  const uint4* s = reinterpret_cast<const uint4*>(pay + uint64_t(b) * pay_stride);
  uint4* d = reinterpret_cast<uint4*>(dst + pos[b]);
  for (uint32_t q = threadIdx.x; q < len / 16; q += blockDim.x) d[q] = s[q];
}

struct Layout {   // workspace layout of gomp_compress_device
  uint64_t src_off, recs_off, meta_off, pos_off, freq_off, lens_off, sb_off, sub_off, pay_off, total;
  uint64_t pay_stride, sub_stride, max_seqs;
};

Layout layout(size_t src_len, const gomp_params* p) {
  Layout L{};
  const uint64_t nb = (uint64_t(src_len) + p->block_size - 1) / p->block_size;
  L.max_seqs = host_max_seqs(p->block_size, p->min_match);
  const uint64_t nsub_max = p->sub_block_seqs ? L.max_seqs / p->sub_block_seqs + 1 : p->sub_blocks_per_block;
  L.sub_stride = 2 * nsub_max;
  L.pay_stride = align16(kTreeBytes + (15ull * p->block_size + 48ull * L.max_seqs) / 8 + 64);
  uint64_t o = 0;
  auto take = [&](uint64_t bytes) { const uint64_t r = o; o = align16(o + bytes) + 256; return r; };
  L.src_off = take(src_len + 64);
  L.recs_off = take(4 * nb * L.max_seqs);
  L.meta_off = take(16 * nb);
  L.pos_off = take(8 * nb);
  if (p->mode == GOMP_MODE_BIT) {
    L.freq_off = take(4 * 316 * nb);
    L.lens_off = take(316 * nb);
    L.sb_off = take(4 * nb);
    L.sub_off = take(4 * L.sub_stride * nb);
    L.pay_off = take(L.pay_stride * nb);
  }
  L.total = o;
  return L;
}

}  // namespace
}  // namespace gomp

using namespace gomp;

GOMP_EXPORT gomp_status gomp_compress_device_workspace_size(size_t src_len, const gomp_params* p, size_t* bytes) {
  if (!bytes || !host_params_ok(p) || p->match_finder != 0 || p->max_chain != 0) return GOMP_ERR_INVALID_ARG;
  *bytes = size_t(layout(src_len, p).total);
  return GOMP_OK;
}

GOMP_EXPORT gomp_status gomp_compress_device(const uint8_t* d_src, size_t src_len, uint8_t* d_dst, size_t dst_cap,
                                             size_t* dst_len, void* d_ws, size_t ws_bytes, const gomp_params* p,
                                             void* stream) {
  if (!dst_len || !d_dst || (!d_src && src_len) || !d_ws || !host_params_ok(p) || p->match_finder != 0 ||
      p->max_chain != 0)
    return GOMP_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(d_dst) | reinterpret_cast<uintptr_t>(d_ws)) & 15u) return GOMP_ERR_INVALID_ARG;
  const Layout Lw = layout(src_len, p);
  if (ws_bytes < Lw.total) return GOMP_ERR_WORKSPACE_TOO_SMALL;
  const uint64_t nb64 = (uint64_t(src_len) + p->block_size - 1) / p->block_size;
  if (nb64 > 0xffffffffull) return GOMP_ERR_INVALID_ARG;
  const uint32_t nb = uint32_t(nb64);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* ws = static_cast<uint8_t*>(d_ws);
  CArgs a{};
  a.src = ws + Lw.src_off;
  a.src_len = src_len;
  a.nb = nb;
  a.block_size = p->block_size;
  a.window = p->window_size;
  a.mm = p->min_match;
  a.maxm = p->max_match;
  a.de = p->de ? 1 : 0;
  a.de_group = p->de ? p->de_group : 0xffffffffu;
  a.max_seqs = uint32_t(Lw.max_seqs);
  uint32_t PR = 1024;   // prev ring: >= window entries, so the positions a chain walk may visit never alias
  while (PR < p->window_size) PR <<= 1;
  a.pm = PR - 1;
  a.recs = reinterpret_cast<uint32_t*>(ws + Lw.recs_off);
  a.meta = reinterpret_cast<uint32_t*>(ws + Lw.meta_off);
  // the input, padded with zeros (word reads past the last byte)
  if (src_len && cudaMemcpyAsync(ws + Lw.src_off, d_src, src_len, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return GOMP_ERR_CUDA;
  if (cudaMemsetAsync(ws + Lw.src_off + src_len, 0, 64, st) != cudaSuccess) return GOMP_ERR_CUDA;
  if (cudaMemsetAsync(a.meta, 0, 16ull * std::max<uint32_t>(nb, 1), st) != cudaSuccess) return GOMP_ERR_CUDA;
  if (nb) {
    const size_t per_warp = ((1u << kHashBits) + 32) * 4 + 2ull * PR;
    const uint32_t nw = uint32_t(std::max<size_t>(1, std::min<size_t>(kParseWarps, (200u << 10) / per_warp)));
    const size_t smem = nw * per_warp;
    cudaFuncSetAttribute(lz_parse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    lz_parse_kernel<<<(nb + nw - 1) / nw, 32 * nw, smem, st>>>(a);
    if (cudaGetLastError() != cudaSuccess) return GOMP_ERR_CUDA;
  }
  std::vector<uint32_t> meta(4ull * nb);
  std::vector<uint32_t> S(nb, 0), nsub(nb, 0);
  std::vector<uint32_t> sub;
  uint64_t* d_pos = reinterpret_cast<uint64_t*>(ws + Lw.pos_off);
  if (p->mode == GOMP_MODE_BIT && nb) {
    uint32_t* d_freq = reinterpret_cast<uint32_t*>(ws + Lw.freq_off);
    freq_kernel<<<nb, kCompThreads, 0, st>>>(a, d_freq);
    // package-merge code lengths and the sub-block size S per block on the device (R14, R12)
    pm_kernel<<<nb, 96, 0, st>>>(a, d_freq, ws + Lw.lens_off, reinterpret_cast<uint32_t*>(ws + Lw.sb_off), p->cwl,
                                 p->sub_block_seqs, p->sub_blocks_per_block);
    if (cudaGetLastError() != cudaSuccess) return GOMP_ERR_CUDA;
    uint8_t* d_lens = ws + Lw.lens_off;
    uint32_t* d_S = reinterpret_cast<uint32_t*>(ws + Lw.sb_off);
    uint32_t* d_sub = reinterpret_cast<uint32_t*>(ws + Lw.sub_off);
    uint8_t* d_pay = ws + Lw.pay_off;
    if (cudaMemsetAsync(d_sub, 0, 4 * Lw.sub_stride * nb, st) != cudaSuccess ||
        cudaMemsetAsync(d_pay, 0, Lw.pay_stride * nb, st) != cudaSuccess)
      return GOMP_ERR_CUDA;
    huff_encode_kernel<<<nb, kCompThreads, 0, st>>>(a, d_lens, d_pay, Lw.pay_stride, d_sub, uint32_t(Lw.sub_stride), d_S);
    sub.resize(Lw.sub_stride * nb);
    if (cudaMemcpyAsync(sub.data(), d_sub, 4 * sub.size(), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(meta.data(), a.meta, 16ull * nb, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaMemcpyAsync(S.data(), d_S, 4ull * nb, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return GOMP_ERR_CUDA;
    for (uint32_t b = 0; b < nb; ++b) {
      nsub[b] = (meta[4 * b] + S[b] - 1) / S[b];
      if (2ull * nsub[b] > Lw.sub_stride) return GOMP_ERR_INVALID_ARG;   // cannot happen: sub_stride bounds it
    }
  } else if (nb) {
    if (cudaMemcpyAsync(meta.data(), a.meta, 16ull * nb, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return GOMP_ERR_CUDA;
  }
  // file layout (FORMAT.md §1), as gomp_compress writes it
  uint64_t n_sub_total = 0, max_tok = 0;
  for (uint32_t b = 0; b < nb; ++b) {
    n_sub_total += nsub[b];
    max_tok = std::max<uint64_t>(max_tok, 4ull * meta[4 * b] + meta[4 * b + 1]);
    meta[4 * b + 3] = uint32_t(p->mode == GOMP_MODE_BIT ? align16(kTreeBytes + (uint64_t(meta[4 * b + 2]) + 7) / 8)
                                                        : align16(4ull * meta[4 * b] + meta[4 * b + 1]));
  }
  if (n_sub_total > 0xffffffffull) return GOMP_ERR_INVALID_ARG;
  const uint64_t base = align16(kHeaderBytes + uint64_t(kBlockEntryBytes) * nb + uint64_t(kSubEntryBytes) * n_sub_total);
  std::vector<uint64_t> pos(nb);
  uint64_t total = base;
  for (uint32_t b = 0; b < nb; ++b) { pos[b] = total; total += meta[4 * b + 3]; }
  total += kTrailerBytes;
  if (total > dst_cap) return GOMP_ERR_DST_TOO_SMALL;
  std::vector<uint8_t> hdr(base, 0);
  uint32_t sub_at = 0;
  for (uint32_t b = 0; b < nb; ++b) {
    uint8_t* e = hdr.data() + kHeaderBytes + uint64_t(kBlockEntryBytes) * b;
    st64(e, pos[b]);
    st32(e + 8, meta[4 * b + 3]);
    st32(e + 12, meta[4 * b]);
    st32(e + 16, meta[4 * b + 1]);
    st32(e + 20, p->mode == GOMP_MODE_BIT ? sub_at : 0);
    st32(e + 24, S[b]);
    st32(e + 28, nsub[b]);
    for (uint32_t k = 0; k < nsub[b]; ++k) {
      uint8_t* s = hdr.data() + kHeaderBytes + uint64_t(kBlockEntryBytes) * nb + uint64_t(kSubEntryBytes) * (sub_at + k);
      st32(s, sub[Lw.sub_stride * b + 2 * k]);
      st32(s + 4, sub[Lw.sub_stride * b + 2 * k + 1]);
    }
    sub_at += nsub[b];
  }
  host_write_header(hdr.data(), p, nb, src_len, total, n_sub_total, max_tok, base);
  if (cudaMemcpyAsync(d_dst, hdr.data(), base, cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaMemcpyAsync(d_pos, pos.data(), 8ull * nb, cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaMemcpyAsync(a.meta, meta.data(), 16ull * nb, cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaMemsetAsync(d_dst + total - kTrailerBytes, 0, kTrailerBytes, st) != cudaSuccess)
    return GOMP_ERR_CUDA;
  if (nb) {
    if (p->mode == GOMP_MODE_BIT) place_kernel<<<nb, 256, 0, st>>>(ws + Lw.pay_off, Lw.pay_stride, a.meta, d_pos, d_dst);
    else byte_payload_kernel<<<nb, kCompThreads, 0, st>>>(a, d_dst, d_pos);
  }
  if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess) return GOMP_ERR_CUDA;
  *dst_len = size_t(total);
  return GOMP_OK;
}
