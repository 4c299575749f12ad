"""Test helper: hand-build Gompresso/Byte files from explicit sequence lists (FORMAT.md §1-§3), and corrupt
files in controlled ways. Independent of both the oracle and the product (used to feed both)."""
import struct

import numpy as np


def byte_file(blocks, block_size, min_match=4, max_match=64, window=8192, de=False):
    """blocks: list of (sequences, literal_bytes); sequences = [(lit_len, L, dist), ...]."""
    nb = len(blocks)
    total = 0
    for seqs, _ in blocks:
        total += sum(l + L for l, L, _ in seqs)
    payload_base = (64 + 32 * nb + 15) & ~15
    body = bytearray()
    table = bytearray()
    pos = payload_base
    for seqs, lits in blocks:
        rec = bytearray()
        for l, L, d in seqs:
            mcode = L - min_match + 1 if L else 0
            rec += struct.pack("<I", l | (mcode << 10) | (((d - 1) if L else 0) << 16))
        p = bytes(rec) + bytes(lits)
        p += b"\0" * ((-len(p)) % 16)
        table += struct.pack("<QIIIIII", pos, len(p), len(seqs), len(lits), 0, 0, 0)
        body += p
        pos += len(p)
    body += b"\0" * 16
    file_len = payload_base + len(body)
    hdr = b"GMPR" + bytes([1, 0, 1 if de else 0, min_match, max_match, 0, 32, 0])
    hdr += struct.pack("<IIIQQIIQII", block_size, window, nb, total, file_len, 0, 0, payload_base, 0, 0)
    assert len(hdr) == 64
    f = hdr + bytes(table)
    f += b"\0" * (payload_base - len(f))
    return np.frombuffer(f + bytes(body), dtype=np.uint8).copy()


def expand(seqs, lits):
    """Sequential expansion, written out (for the hand-built cases)."""
    out = bytearray()
    lp = 0
    for l, L, d in seqs:
        out += lits[lp: lp + l]
        lp += l
        for _ in range(L):
            out.append(out[-d])
    return bytes(out)
