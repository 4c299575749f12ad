// api.cpp — host-only C-ABI entry points of libgompresso.so: header parsing, table validation, workspace
// sizing, multi-GPU shard planning, status strings. The device entry points live in decode.cu.
#include <algorithm>
#include <cstdint>
#include <cstring>

#include "format.hpp"
#include "gomp.h"

using namespace gomp;

#define GOMP_EXPORT extern "C" __attribute__((visibility("default")))

GOMP_EXPORT int gomp_version(void) { return GOMP_ABI_VERSION; }

GOMP_EXPORT const char* gomp_status_string(gomp_status s) {
  switch (s) {
    case GOMP_OK: return "OK";
    case GOMP_ERR_INVALID_ARG: return "INVALID_ARG";
    case GOMP_ERR_BAD_MAGIC: return "BAD_MAGIC";
    case GOMP_ERR_UNSUPPORTED_VERSION: return "UNSUPPORTED_VERSION";
    case GOMP_ERR_TRUNCATED: return "TRUNCATED";
    case GOMP_ERR_HEADER_INCONSISTENT: return "HEADER_INCONSISTENT";
    case GOMP_ERR_CORRUPT_STREAM: return "CORRUPT_STREAM";
    case GOMP_ERR_MALFORMED_BACKREF: return "MALFORMED_BACKREF";
    case GOMP_ERR_NO_PROGRESS: return "NO_PROGRESS";
    case GOMP_ERR_DST_TOO_SMALL: return "DST_TOO_SMALL";
    case GOMP_ERR_WORKSPACE_TOO_SMALL: return "WORKSPACE_TOO_SMALL";
    case GOMP_ERR_CUDA: return "CUDA";
    case GOMP_ERR_OOM: return "OOM";
  }
  return "UNKNOWN";
}

GOMP_EXPORT gomp_status gomp_get_info(const uint8_t* hdr, size_t hdr_len, gomp_info* out) {
  return parse_header(hdr, hdr_len, out);
}

GOMP_EXPORT gomp_status gomp_validate_tables(const uint8_t* f, size_t len, uint32_t* bad_block) {
  gomp_info in;
  if (bad_block) *bad_block = 0;
  gomp_status st = parse_header(f, len, &in);
  if (st != GOMP_OK) return st;
  if (in.file_len > len) return GOMP_ERR_TRUNCATED;
  uint64_t sub_at = 0, max_tok = 0;
  for (uint32_t b = 0; b < in.n_blocks; ++b) {
    BlockEntry e;
    std::memcpy(&e, f + kHeaderBytes + uint64_t(kBlockEntryBytes) * b, sizeof(e));
    bool ok = e.payload_off % 16 == 0 && e.payload_len % 16 == 0 && e.payload_off >= in.payload_base &&
              e.payload_off + e.payload_len <= in.file_len - kTrailerBytes;
    const uint64_t ulen = std::min<uint64_t>(in.block_size, in.uncompressed_len - uint64_t(b) * in.block_size);
    ok = ok && e.n_lit <= ulen && e.n_seq <= ulen && (e.n_seq > 0) == (ulen > 0);
    if (in.mode == GOMP_MODE_BYTE) {
      ok = ok && e.sub_first == 0 && e.S == 0 && e.n_sub == 0 && 4ull * e.n_seq + e.n_lit <= e.payload_len;
    } else {
      ok = ok && e.S >= 1 && e.n_sub == (e.n_seq + e.S - 1) / e.S && e.sub_first == sub_at &&
           e.payload_len >= kTreeBytes;
      uint64_t bits = 0, lits = 0;
      if (ok && sub_at + e.n_sub <= in.n_sub_total) {
        for (uint32_t k = 0; k < e.n_sub; ++k) {
          const uint8_t* s = f + kHeaderBytes + uint64_t(kBlockEntryBytes) * in.n_blocks + uint64_t(kSubEntryBytes) * (sub_at + k);
          bits += ld32(s);
          lits += ld32(s + 4);
        }
        ok = lits == e.n_lit && (bits + 7) / 8 <= uint64_t(e.payload_len) - kTreeBytes;
      } else {
        ok = false;
      }
      sub_at += e.n_sub;
      max_tok = std::max<uint64_t>(max_tok, 4ull * e.n_seq + e.n_lit);
    }
    if (!ok) {
      if (bad_block) *bad_block = b;
      return GOMP_ERR_HEADER_INCONSISTENT;
    }
  }
  if (in.mode == GOMP_MODE_BIT && (sub_at != in.n_sub_total || max_tok != in.max_block_tokens))
    return GOMP_ERR_HEADER_INCONSISTENT;
  return GOMP_OK;
}

GOMP_EXPORT gomp_status gomp_decompress_workspace_size(const gomp_info* info, uint32_t n_blocks, size_t* bytes) {
  if (!info || !bytes) return GOMP_ERR_INVALID_ARG;
  const uint64_t nb = n_blocks ? n_blocks : info->n_blocks;
  uint64_t ws = kWsHeaderBytes;
  if (info->mode == GOMP_MODE_BIT) ws += nb * align16(info->max_block_tokens) + 64;
  *bytes = size_t(ws);
  return GOMP_OK;
}

GOMP_EXPORT gomp_status gomp_plan_shards(const uint8_t* f, size_t len, int n_dev, uint32_t* first_block) {
  gomp_info in;
  if (!first_block || n_dev < 1) return GOMP_ERR_INVALID_ARG;
  gomp_status st = parse_header(f, len, &in);
  if (st != GOMP_OK) return st;
  if (len < kHeaderBytes + uint64_t(kBlockEntryBytes) * in.n_blocks) return GOMP_ERR_TRUNCATED;
  uint64_t total = 0;
  for (uint32_t b = 0; b < in.n_blocks; ++b) total += ld32(f + kHeaderBytes + uint64_t(kBlockEntryBytes) * b + 8);
  // boundary d = first block whose cumulative compressed bytes reach d/n_dev of the total
  first_block[0] = 0;
  uint64_t acc = 0;
  uint32_t b = 0;
  for (int d = 1; d < n_dev; ++d) {
    const uint64_t target = total * uint64_t(d) / uint64_t(n_dev);
    while (b < in.n_blocks && acc + ld32(f + kHeaderBytes + uint64_t(kBlockEntryBytes) * b + 8) / 2 <= target) {
      acc += ld32(f + kHeaderBytes + uint64_t(kBlockEntryBytes) * b + 8);
      ++b;
    }
    first_block[d] = b;
  }
  first_block[n_dev] = in.n_blocks;
  return GOMP_OK;
}

// Standalone file of blocks [first, first + n): header with the shard's block count and length,
// the block entries with payload offsets and sub-table indices rebased, the shard's sub-table entries, and the
// payloads packed in block order (16-byte aligned), so a device holds O(shard) bytes instead of the whole file.
GOMP_EXPORT gomp_status gomp_shard_file(const uint8_t* f, size_t len, uint32_t first, uint32_t n, uint8_t* out,
                                        size_t cap, size_t* out_len) {
  gomp_info in;
  if (!out_len) return GOMP_ERR_INVALID_ARG;
  gomp_status st = parse_header(f, len, &in);
  if (st != GOMP_OK) return st;
  if (uint64_t(first) + n > in.n_blocks) return GOMP_ERR_INVALID_ARG;
  if (len < in.payload_base) return GOMP_ERR_TRUNCATED;
  const bool bit = in.mode == GOMP_MODE_BIT;
  uint64_t n_sub = 0, pay = 0, max_tok = 0;
  for (uint32_t b = first; b < first + n; ++b) {
    BlockEntry e;
    std::memcpy(&e, f + kHeaderBytes + uint64_t(kBlockEntryBytes) * b, sizeof(e));
    if (e.payload_off % 16 || e.payload_len % 16 || e.payload_off < in.payload_base ||
        e.payload_off + e.payload_len > std::min<uint64_t>(len, in.file_len)) return GOMP_ERR_HEADER_INCONSISTENT;
    if (bit && uint64_t(e.sub_first) + e.n_sub > in.n_sub_total) return GOMP_ERR_HEADER_INCONSISTENT;
    n_sub += bit ? e.n_sub : 0;
    pay += e.payload_len;
    max_tok = std::max<uint64_t>(max_tok, 4ull * e.n_seq + e.n_lit);
  }
  const uint64_t total_lo = uint64_t(first) * in.block_size;
  const uint64_t total = std::min<uint64_t>(uint64_t(first + n) * in.block_size, in.uncompressed_len) -
                         std::min<uint64_t>(total_lo, in.uncompressed_len);
  const uint64_t base = align16(kHeaderBytes + uint64_t(kBlockEntryBytes) * n + uint64_t(kSubEntryBytes) * n_sub);
  const uint64_t flen = base + pay + kTrailerBytes;
  *out_len = size_t(flen);
  if (!out) return GOMP_OK;                 // size query
  if (cap < flen) return GOMP_ERR_DST_TOO_SMALL;
  std::memset(out, 0, size_t(base));
  std::memcpy(out, f, kHeaderBytes);
  st32(out + 20, n);
  st64(out + 24, total);
  st64(out + 32, flen);
  st32(out + 40, uint32_t(n_sub));
  st32(out + 44, bit ? uint32_t(max_tok) : 0u);
  st64(out + 48, base);
  uint64_t at = base, sub_at = 0;
  for (uint32_t i = 0; i < n; ++i) {
    BlockEntry e;
    std::memcpy(&e, f + kHeaderBytes + uint64_t(kBlockEntryBytes) * (first + i), sizeof(e));
    std::memcpy(out + at, f + e.payload_off, e.payload_len);
    if (bit) {
      std::memcpy(out + kHeaderBytes + uint64_t(kBlockEntryBytes) * n + uint64_t(kSubEntryBytes) * sub_at,
                  f + kHeaderBytes + uint64_t(kBlockEntryBytes) * in.n_blocks + uint64_t(kSubEntryBytes) * e.sub_first,
                  uint64_t(kSubEntryBytes) * e.n_sub);
      e.sub_first = uint32_t(sub_at);
      sub_at += e.n_sub;
    }
    e.payload_off = at;
    std::memcpy(out + kHeaderBytes + uint64_t(kBlockEntryBytes) * i, &e, sizeof(e));
    at += e.payload_len;
  }
  std::memset(out + at, 0, kTrailerBytes);
  return GOMP_OK;
}
