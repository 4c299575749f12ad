"""Test helper (not an oracle): wrap one Gompresso/Bit block in a raw-DEFLATE dynamic block so that stock
zlib can inflate it. This pins the Bit symbol layer (canonical codes of RFC 1951 §3.2.2, LSB-first packing of
§3.1.1, length/distance codes and extra bits of §3.2.5, EOB) against an implementation we did not write.

The 160-byte Gompresso tree header (286 + 30 nibbles, FORMAT.md §3) is replaced by an RFC 1951 §3.2.7
dynamic header: HLIT=286, HDIST=30, HCLEN=19 with every code-length symbol 0..15 given a 4-bit code (a complete
code; 16/17/18 unused), then the 316 code lengths, then the block's bit-concatenated sub-blocks.
"""
import struct

CL_ORDER = [16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15]


class BitWriter:
    def __init__(self):
        self.v = 0
        self.n = 0

    def put(self, value, nbits):  # integer LSB-first
        self.v |= (value & ((1 << nbits) - 1)) << self.n
        self.n += nbits

    def put_code(self, code, length):  # Huffman code, MSB-first
        for i in range(length - 1, -1, -1):
            self.put((code >> i) & 1, 1)

    def put_bits_from(self, data: bytes, nbits):
        self.v |= (int.from_bytes(data, "little") & ((1 << nbits) - 1)) << self.n
        self.n += nbits

    def bytes(self):
        return self.v.to_bytes((self.n + 7) // 8, "little")


def block_to_deflate(f: bytes, b: int) -> bytes:
    """Raw DEFLATE stream (one final dynamic block) for block b of a Gompresso/Bit file f."""
    nb = struct.unpack_from("<I", f, 20)[0]
    off, plen, n_seq, n_lit, sub_first, S, n_sub = struct.unpack_from("<QIIIIII", f, 64 + 32 * b)
    pl = f[off: off + plen]
    llen = [(pl[i // 2] >> (4 * (i & 1))) & 15 for i in range(286)]
    dlen = [(pl[143 + i // 2] >> (4 * (i & 1))) & 15 for i in range(30)]
    bits = 0
    for k in range(n_sub):
        bits += struct.unpack_from("<I", f, 64 + 32 * nb + 8 * (sub_first + k))[0]
    w = BitWriter()
    w.put(1, 1)          # BFINAL
    w.put(2, 2)          # BTYPE = 10 (dynamic)
    w.put(286 - 257, 5)  # HLIT
    w.put(30 - 1, 5)     # HDIST
    w.put(19 - 4, 4)     # HCLEN
    cl_len = {s: (4 if s <= 15 else 0) for s in range(19)}
    for s in CL_ORDER:
        w.put(cl_len[s], 3)
    # canonical code for 16 symbols of length 4: symbol s -> code s
    for ln in llen + dlen:
        w.put_code(ln, 4)
    w.put_bits_from(pl[160:], bits)
    return w.bytes()
