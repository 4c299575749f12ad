"""TEST INFRASTRUCTURE ONLY — ctypes binding of the plain CPU oracle (oracle/oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import this.
The oracle shares no code with paper_1606_00519_b200 (the product). See oracle.c's header for what each
function follows in PAPER.md and which pins in tests/ fix it.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

STATUS = {0: "OK", -1: "INVALID_ARG", -2: "BAD_MAGIC", -3: "UNSUPPORTED_VERSION", -4: "TRUNCATED",
          -5: "HEADER_INCONSISTENT", -6: "CORRUPT_STREAM", -7: "MALFORMED_BACKREF", -8: "NO_PROGRESS",
          -9: "DST_TOO_SMALL"}


class OracleError(Exception):
    def __init__(self, status, block=0):
        super().__init__(f"oracle: {STATUS.get(status, status)} (block {block})")
        self.status = status
        self.name = STATUS.get(status, str(status))
        self.block = block


class Params(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint32) for n in (
        "mode", "de", "block_size", "window_size", "min_match", "max_match", "sub_block_seqs",
        "sub_blocks_per_block", "cwl", "de_group")]


def params(mode="byte", de=True, block_size=262144, window_size=8192, min_match=4, max_match=64,
           sub_block_seqs=16, sub_blocks_per_block=0, cwl=10, de_group=32):
    """Defaults = the paper's setup: 256 KB blocks, 8 KB window, 64-byte lookahead,
    16-sequence sub-blocks, CWL 10; min_match 4 (reading R8)."""
    m = {"byte": 0, "bit": 1}[mode] if isinstance(mode, str) else int(mode)
    return Params(m, int(bool(de)), block_size, window_size, min_match, max_match, sub_block_seqs,
                  sub_blocks_per_block, cwl, de_group)


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError("oracle/liboracle.so missing: run __graft_entry__.build()")
        L = ctypes.CDLL(path)
        P, u8p, u32p, u64p = ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p
        L.or_compress_bound.argtypes = [ctypes.c_uint64, ctypes.POINTER(Params)]
        L.or_compress_bound.restype = ctypes.c_uint64
        L.or_compress.argtypes = [u8p, ctypes.c_uint64, ctypes.POINTER(Params), u8p, ctypes.c_uint64,
                                  ctypes.POINTER(ctypes.c_uint64)]
        L.or_decompress.argtypes = [u8p, ctypes.c_uint64, u8p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64),
                                    ctypes.POINTER(ctypes.c_uint32)]
        L.or_decompress_range.argtypes = [u8p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, u8p,
                                          ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint32)]
        L.or_info.argtypes = [u8p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint32)]
        L.or_block_sequences.argtypes = [u8p, ctypes.c_uint64, ctypes.c_uint32, u32p, u32p, u32p, ctypes.c_uint32,
                                         ctypes.POINTER(ctypes.c_uint32)]
        L.or_parse_block.argtypes = [u8p, ctypes.c_uint32, ctypes.POINTER(Params), u32p, u32p, u32p,
                                     ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint32)]
        L.or_package_merge.argtypes = [u64p, ctypes.c_int, ctypes.c_int, u8p]
        L.or_canonical_codes.argtypes = [u8p, ctypes.c_int, u32p]
        L.or_mrr_simulate.argtypes = [u8p, ctypes.c_uint64, u64p, u64p]
        L.or_mrr_group_rounds.argtypes = [u32p, u32p, u32p, ctypes.c_int, ctypes.c_uint32, u64p, u32p]
        L.or_verify_de.argtypes = [u8p, ctypes.c_uint64]
        for f in ("or_compress", "or_decompress", "or_decompress_range", "or_info", "or_block_sequences",
                  "or_parse_block", "or_package_merge", "or_canonical_codes", "or_mrr_simulate",
                  "or_mrr_group_rounds", "or_verify_de"):
            getattr(L, f).restype = ctypes.c_int
        _LIB = L
    return _LIB


def _u8(x):
    if isinstance(x, (bytes, bytearray)):
        return np.frombuffer(bytes(x), dtype=np.uint8)
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint8))


def compress(data, p=None, **kw):
    """Oracle compressor (greedy exhaustive longest match; FORMAT.md). Returns a numpy uint8 file."""
    src = _u8(data)
    p = p or params(**kw)
    cap = _lib().or_compress_bound(len(src), ctypes.byref(p))
    out = np.empty(int(cap), dtype=np.uint8)
    n = ctypes.c_uint64(0)
    st = _lib().or_compress(src.ctypes.data, len(src), ctypes.byref(p), out.ctypes.data, cap, ctypes.byref(n))
    if st:
        raise OracleError(st)
    return out[: n.value].copy()


def info(f):
    f = _u8(f)
    total, nb = ctypes.c_uint64(0), ctypes.c_uint32(0)
    st = _lib().or_info(f.ctypes.data, len(f), ctypes.byref(total), ctypes.byref(nb))
    if st:
        raise OracleError(st)
    return total.value, nb.value


def decompress(f):
    """The plain definition: sequential expansion of every block's sequences."""
    f = _u8(f)
    total, _ = info(f)
    out = np.empty(max(int(total), 1), dtype=np.uint8)
    n, eb = ctypes.c_uint64(0), ctypes.c_uint32(0)
    st = _lib().or_decompress(f.ctypes.data, len(f), out.ctypes.data, len(out), ctypes.byref(n), ctypes.byref(eb))
    if st:
        raise OracleError(st, eb.value)
    return out[: n.value]


def decompress_blocks(f, b0, b1, block_size):
    """Decompress blocks [b0, b1) only (sampled parity at full size)."""
    f = _u8(f)
    out = np.empty(max((b1 - b0) * block_size, 1), dtype=np.uint8)
    eb = ctypes.c_uint32(0)
    st = _lib().or_decompress_range(f.ctypes.data, len(f), b0, b1, out.ctypes.data, len(out), ctypes.byref(eb))
    if st:
        raise OracleError(st, eb.value)
    total, nb = info(f)
    end = min(b1 * block_size, total)
    return out[: end - b0 * block_size]


def block_sequences(f, b, cap=1 << 20):
    f = _u8(f)
    a = np.zeros((3, cap), dtype=np.uint32)
    n = ctypes.c_uint32(0)
    st = _lib().or_block_sequences(f.ctypes.data, len(f), b, a[0].ctypes.data, a[1].ctypes.data, a[2].ctypes.data,
                                   cap, ctypes.byref(n))
    if st:
        raise OracleError(st, b)
    return [tuple(int(v) for v in a[:, i]) for i in range(n.value)]


def parse_block(data, p=None, **kw):
    """Greedy (DE-aware) parse of one raw block: list of (lit_len, L, dist)."""
    src = _u8(data)
    p = p or params(**kw)
    cap = len(src) + 2
    a = np.zeros((3, cap), dtype=np.uint32)
    n = ctypes.c_uint32(0)
    st = _lib().or_parse_block(src.ctypes.data, len(src), ctypes.byref(p), a[0].ctypes.data, a[1].ctypes.data,
                               a[2].ctypes.data, cap, ctypes.byref(n))
    if st:
        raise OracleError(st)
    return [tuple(int(v) for v in a[:, i]) for i in range(n.value)]


def package_merge(freq, maxlen):
    fr = np.ascontiguousarray(np.asarray(freq, dtype=np.uint64))
    lens = np.zeros(len(fr), dtype=np.uint8)
    st = _lib().or_package_merge(fr.ctypes.data, len(fr), maxlen, lens.ctypes.data)
    if st:
        raise OracleError(st)
    return [int(x) for x in lens]


def canonical_codes(lens):
    ln = np.ascontiguousarray(np.asarray(lens, dtype=np.uint8))
    codes = np.zeros(len(ln), dtype=np.uint32)
    st = _lib().or_canonical_codes(ln.ctypes.data, len(ln), codes.ctypes.data)
    if st:
        raise OracleError(st)
    return [int(x) for x in codes]


def mrr_simulate(f):
    """Rounds histogram hist[r] (groups needing r MRR rounds) and bytes copied per round (R1, R20)."""
    f = _u8(f)
    hist = np.zeros(33, dtype=np.uint64)
    nbytes = np.zeros(33, dtype=np.uint64)
    st = _lib().or_mrr_simulate(f.ctypes.data, len(f), hist.ctypes.data, nbytes.ctypes.data)
    if st:
        raise OracleError(st)
    return hist, nbytes


def mrr_group(seqs, o0=0):
    """MRR on one explicit group [(lit_len, L, dist), ...]: (rounds, round_of_lane, bytes_per_round)."""
    n = len(seqs)
    a = np.zeros((3, 32), dtype=np.uint32)
    for i, (l, L, d) in enumerate(seqs):
        a[:, i] = (l, L, d)
    br = np.zeros(33, dtype=np.uint64)
    rl = np.zeros(32, dtype=np.uint32)
    r = _lib().or_mrr_group_rounds(a[0].ctypes.data, a[1].ctypes.data, a[2].ctypes.data, n, o0, br.ctypes.data,
                                   rl.ctypes.data)
    if r < 0:
        raise OracleError(r)
    return r, [int(x) for x in rl[:n]], [int(x) for x in br]


def verify_de(f):
    f = _u8(f)
    r = _lib().or_verify_de(f.ctypes.data, len(f))
    if r < 0:
        raise OracleError(r)
    return bool(r)
