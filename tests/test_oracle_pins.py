"""Pins of the CPU oracle against things other than itself (CPU only, `-m "not gpu"`).

Each test names what fixes the oracle: a value printed in the paper, a textbook example, a stock library
(zlib) that we did not write, a closed form / invariant, or brute force on tiny inputs.
"""
import heapq
import itertools
import json
import os
import zlib

import numpy as np
import pytest

import datagen
import oracle
from deflate_pin import block_to_deflate
from fmt_util import byte_file, expand

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


# ---------------------------------------------------------------- round trip
CASES = [
    ("text", 70_000), ("wiki", 90_000), ("matrix", 80_000), ("random", 20_000), ("zeros", 50_000),
    ("nested8", 40_000),
]


def _data(kind, n, seed=1):
    if kind == "zeros":
        return datagen.zeros(n)
    if kind.startswith("nested"):
        return datagen.nested(n, int(kind[6:]), seed=seed)
    return datagen.GENERATORS[kind](n, seed=seed)


@pytest.mark.parametrize("kind,n", CASES)
@pytest.mark.parametrize("mode", ["byte", "bit"])
@pytest.mark.parametrize("de", [True, False])
def test_round_trip(kind, n, mode, de):
    x = _data(kind, n)
    c = oracle.compress(x, mode=mode, de=de, block_size=32768, sub_block_seqs=16 if mode == "bit" else 0)
    assert np.array_equal(oracle.decompress(c), x)
    if de:
        assert oracle.verify_de(c)


@pytest.mark.parametrize("n", [0, 1, 15, 16, 17, 4095, 4096, 4097, 12289])
@pytest.mark.parametrize("mode", ["byte", "bit"])
def test_round_trip_edges(n, mode):
    x = datagen.text(n, seed=3)
    c = oracle.compress(x, mode=mode, block_size=4096, sub_block_seqs=0, sub_blocks_per_block=3)
    assert np.array_equal(oracle.decompress(c), x)


@pytest.mark.parametrize("mode", ["byte", "bit"])
def test_literal_run_cap(mode):
    """R10: literal runs close at exactly 1023 bytes (literal-only sequence)."""
    x = datagen.random_bytes(3000, seed=9)
    c = oracle.compress(x, mode=mode, block_size=4096, sub_block_seqs=2)
    seqs = oracle.block_sequences(c, 0)
    assert [s[0] for s in seqs] == [1023, 1023, 954]
    assert all(s[1] == 0 for s in seqs)
    assert np.array_equal(oracle.decompress(c), x)


def test_min_match_3_and_params():
    x = datagen.wiki(30_000, seed=4)
    for mm, mx, w in [(3, 65, 32768), (4, 66, 1), (4, 4, 100), (3, 258 - 255 + 3, 8192)]:
        c = oracle.compress(x, mode="bit", min_match=mm, max_match=mx, window_size=w, block_size=16384,
                            sub_block_seqs=7)
        assert np.array_equal(oracle.decompress(c), x)
        for b in range(2):
            for l, L, d in oracle.block_sequences(c, b):
                assert L == 0 or (mm <= L <= mx and L <= d <= w)


# ---------------------------------------------------------------- the paper's worked LZ77 example
def test_paper_fig_example():
    g = gold("fig_example.json")
    seqs = oracle.parse_block(g["input"].encode(), min_match=g["min_match"], de=False)
    assert [list(s) for s in seqs] == g["expected_sequences"]
    # with the default min_match = 4 the same input has no back-reference (R8)
    assert oracle.parse_block(g["input"].encode(), de=False) == [(7, 0, 0)]


# ---------------------------------------------------------------- brute-force greedy parse on tiny inputs
def _brute_best(x, c, ls, hwm, p):
    """Enumerate every source s and every length by direct slice comparison; DE admissibility of
    FORMAT.md §4 (R4/R5); longest wins, ties to the smallest distance (R7)."""
    best = (0, 0)
    for s in range(max(0, c - p["window"]), c):
        for L in range(min(p["max"], len(x) - c, c - s), 0, -1):
            if p["de"] and s < ls:
                if not (s + L <= hwm):
                    continue
            if x[s:s + L] == x[c:c + L]:
                if L > best[0] or (L == best[0] and c - s < best[1]):
                    best = (L, c - s)
                break
    return best


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("de,group", [(False, 32), (True, 32), (True, 64), (True, 128)])
def test_parse_is_greedy_longest(seed, de, group):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(40, 220)) if group == 32 else int(rng.integers(24 * group, 30 * group))
    x = bytes(rng.choice(np.frombuffer(b"abc", np.uint8), size=n, p=[0.6, 0.3, 0.1]))
    p = dict(window=int(rng.integers(4, 40)), max=int(rng.integers(4, 12)), de=de, mm=3)
    seqs = oracle.parse_block(x, min_match=3, max_match=p["max"], window_size=p["window"], de=de, de_group=group)
    c = 0
    hwm = 0
    for i, (l, L, d) in enumerate(seqs):
        ls = c
        for k in range(l):  # every literal position: no admissible candidate of length >= min_match
            best = _brute_best(x, c, ls, hwm, p)
            assert best[0] < p["mm"], (i, c, best)
            c += 1
        if L:
            assert _brute_best(x, c, ls, hwm, p) == (L, d)
            c += L
        if (i + 1) % group == 0:   # warpHWM <- pos after every de_group-th sequence
            hwm = c
    assert c == len(x)
    if group > 32:
        assert len(seqs) > 2 * group, "the input must span several DE groups"
    assert expand(seqs, _literals(x, seqs)) == x


def _literals(x, seqs):
    out = bytearray()
    c = 0
    for l, L, _ in seqs:
        out += x[c:c + l]
        c += l + L
    return bytes(out)


# ---------------------------------------------------------------- canonical codes: RFC 1951 §3.2.2 example
def test_rfc1951_canonical_example():
    g = gold("rfc1951_canonical.json")
    codes = oracle.canonical_codes(g["lengths"])
    got = [format(c, f"0{ln}b") for c, ln in zip(codes, g["lengths"])]
    assert got == g["codes"]


# ---------------------------------------------------------------- package-merge: Kraft, optimality
def _huffman_cost(freq):
    h = [f for f in freq if f]
    if len(h) < 2:
        return sum(h)
    heapq.heapify(h)
    cost = 0
    while len(h) > 1:
        a, b = heapq.heappop(h), heapq.heappop(h)
        cost += a + b
        heapq.heappush(h, a + b)
    return cost


def _huffman_maxlen(freq):
    items = [(f, i, 0) for i, f in enumerate(freq) if f]
    depth = {i: 0 for _, i, _ in items}
    members = {i: [i] for _, i, _ in items}
    h = [(f, i) for f, i, _ in items]
    heapq.heapify(h)
    nxt = len(freq)
    while len(h) > 1:
        (fa, a), (fb, b) = heapq.heappop(h), heapq.heappop(h)
        members[nxt] = members.pop(a) + members.pop(b)
        for m in members[nxt]:
            depth[m] += 1
        heapq.heappush(h, (fa + fb, nxt))
        nxt += 1
    return max(depth.values()) if depth else 0


@pytest.mark.parametrize("seed", range(30))
def test_package_merge_optimal_small(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 7))
    maxlen = int(rng.integers(max(1, int(np.ceil(np.log2(n)))), 5))
    freq = [int(v) for v in rng.integers(1, 50, size=n)]
    lens = oracle.package_merge(freq, maxlen)
    assert sum(2.0 ** -l for l in lens) == 1.0 and max(lens) <= maxlen
    best = min(sum(f * l for f, l in zip(freq, ls))
               for ls in itertools.product(range(1, maxlen + 1), repeat=n) if sum(2.0 ** -l for l in ls) <= 1)
    assert sum(f * l for f, l in zip(freq, lens)) == best


@pytest.mark.parametrize("seed", range(10))
def test_package_merge_large(seed):
    rng = np.random.default_rng(100 + seed)
    n = 286
    freq = [int(v) for v in (rng.zipf(1.3, size=n) * (rng.random(n) < 0.8))]
    lens = oracle.package_merge(freq, 10)
    used = [l for f, l in zip(freq, lens) if f]
    assert all((l > 0) == (f > 0) for f, l in zip(freq, lens))
    assert max(used) <= 10
    assert sum(2.0 ** -l for l in used) == 1.0
    if _huffman_maxlen(freq) <= 10:  # unconstrained Huffman fits: same cost
        assert sum(f * l for f, l in zip(freq, lens)) == _huffman_cost(freq)
    else:  # constraint binds: cost >= Huffman
        assert sum(f * l for f, l in zip(freq, lens)) >= _huffman_cost(freq)


def test_package_merge_degenerate():
    assert oracle.package_merge([0, 0, 5, 0], 10) == [0, 0, 1, 0]
    assert oracle.package_merge([0, 0, 0], 10) == [0, 0, 0]
    assert oracle.package_merge([1, 1], 10) == [1, 1]
    assert oracle.package_merge([1, 1, 1, 1], 2) == [2, 2, 2, 2]


# ---------------------------------------------------------------- Bit symbol layer: stock zlib inflate
@pytest.mark.parametrize("kind", ["wiki", "matrix", "random", "zeros", "nested4"])
@pytest.mark.parametrize("de", [True, False])
def test_bit_blocks_inflate_with_zlib(kind, de):
    x = _data(kind, 50_000, seed=5)
    bs = 16384
    c = oracle.compress(x, mode="bit", de=de, block_size=bs, sub_block_seqs=0, sub_blocks_per_block=5)
    cb = bytes(c)
    nb = (len(x) + bs - 1) // bs
    for b in range(nb):
        raw = zlib.decompressobj(-15).decompress(block_to_deflate(cb, b))
        assert raw == bytes(x[b * bs:(b + 1) * bs]), b


# ---------------------------------------------------------------- Bit <-> Byte: same parse, same records
@pytest.mark.parametrize("kind", ["wiki", "matrix", "nested16"])
def test_bit_and_byte_same_sequences(kind):
    x = _data(kind, 40_000, seed=6)
    cb = oracle.compress(x, mode="byte", block_size=16384)
    ct = oracle.compress(x, mode="bit", block_size=16384, sub_block_seqs=16)
    for b in range(3):
        assert oracle.block_sequences(cb, b) == oracle.block_sequences(ct, b)


def test_sub_block_table_sums():
    import struct
    x = datagen.wiki(60_000, seed=8)
    c = bytes(oracle.compress(x, mode="bit", block_size=32768, sub_block_seqs=0, sub_blocks_per_block=16))
    nb = struct.unpack_from("<I", c, 20)[0]
    for b in range(nb):
        off, plen, n_seq, n_lit, sf, S, ns = struct.unpack_from("<QIIIIII", c, 64 + 32 * b)
        subs = [struct.unpack_from("<II", c, 64 + 32 * nb + 8 * (sf + k)) for k in range(ns)]
        assert ns == 16 or ns == -(-n_seq // S)
        assert sum(s[1] for s in subs) == n_lit
        assert (sum(s[0] for s in subs) + 7) // 8 + 160 <= plen


# ---------------------------------------------------------------- MRR (Fig. alg:mrr) examples and invariants
def test_mrr_paper_example():
    g = gold("mrr_examples.json")["paper_three_sequences"]
    r, lanes, _ = oracle.mrr_group([tuple(s) for s in g["group"]])
    assert r == g["rounds"] and lanes == g["round_of_lane"]


def test_mrr_adversarial_chain():
    g = gold("mrr_examples.json")["adversarial_chain"]
    seqs = [tuple(s) for s in g["group"]]
    r, lanes, _ = oracle.mrr_group(seqs)
    assert r == g["rounds"] and lanes == g["round_of_lane"]
    f = byte_file([(seqs, g["literals"].encode())], block_size=64)
    assert bytes(oracle.decompress(f)) == g["output"].encode()
    h, nbytes = oracle.mrr_simulate(f)
    assert h[3] == 1 and list(nbytes[1:4]) == [8, 8, 8]


def test_ballot_definition():
    g = gold("mrr_examples.json")["ballot"]
    assert sum(1 << i for i in g["votes_lanes"]) == g["value"]


@pytest.mark.parametrize("depth", [1, 2, 4, 8, 16, 32])
def test_nesting_depth_point_mass(depth):
    """one repeated string -> 32 rounds, two -> 16, four -> 8 ...; DE -> 1 round."""
    x = datagen.nested(40_000, depth, seed=3)
    c = oracle.compress(x, mode="byte", de=False, block_size=40_000)
    h, _ = oracle.mrr_simulate(c)
    groups = int(h.sum())
    assert h[depth] >= groups - 3, {i: int(v) for i, v in enumerate(h) if v}
    assert h[max(depth, 2) + 1:].sum() == 0  # boundary groups may differ by one round, never exceed D
    cd = oracle.compress(x, mode="byte", de=True, block_size=40_000)
    hd, _ = oracle.mrr_simulate(cd)
    assert hd[2:].sum() == 0 and oracle.verify_de(cd)
    if depth > 1:
        assert not oracle.verify_de(c)


@pytest.mark.parametrize("kind", ["wiki", "matrix"])
def test_mrr_progress_on_real_shaped_data(kind):
    x = _data(kind, 65536, seed=2)
    c = oracle.compress(x, mode="byte", de=False, block_size=65536)
    h, nbytes = oracle.mrr_simulate(c)  # raises NO_PROGRESS if a round copied nothing
    assert h.sum() > 0 and nbytes[1] > 0
    cd = oracle.compress(x, mode="byte", de=True, block_size=65536)
    hd, _ = oracle.mrr_simulate(cd)
    assert hd[2:].sum() == 0


# ---------------------------------------------------------------- validation / error paths
def _expect(status, f):
    with pytest.raises(oracle.OracleError) as e:
        oracle.decompress(f)
    assert e.value.name == status


def test_errors():
    x = datagen.text(20_000, seed=2)
    c = oracle.compress(x, mode="byte", block_size=8192)
    bad = c.copy(); bad[0] = ord("X"); _expect("BAD_MAGIC", bad)
    bad = c.copy(); bad[4] = 2; _expect("UNSUPPORTED_VERSION", bad)
    _expect("TRUNCATED", c[:40])
    _expect("TRUNCATED", c[:-1])
    bad = c.copy(); bad[20] += 1; _expect("HEADER_INCONSISTENT", bad)
    # overlapping back-reference (dist < L) is malformed (R2)
    f = byte_file([([(4, 4, 2)], b"abcd")], block_size=16)
    _expect("MALFORMED_BACKREF", f)
    # reference before the block start (R9)
    f = byte_file([([(2, 4, 5)], b"ab")], block_size=16)
    _expect("MALFORMED_BACKREF", f)
    # beyond the window
    f = byte_file([([(16, 0, 0)], b"a" * 16), ([(8, 4, 8), (0, 4, 12)], b"b" * 8)], block_size=16, window=8)
    _expect("MALFORMED_BACKREF", f)
    # sizes that do not add up to the block length
    f = byte_file([([(3, 0, 0)], b"abc")], block_size=16)
    f[24] = 4  # uncompressed_len 4 != 3
    _expect("CORRUPT_STREAM", f)


def test_bit_corruption_detected():
    x = datagen.wiki(40_000, seed=2)
    c = oracle.compress(x, mode="bit", block_size=16384, sub_block_seqs=0, sub_blocks_per_block=4)
    rng = np.random.default_rng(0)
    import struct
    off = struct.unpack_from("<Q", bytes(c), 64)[0]
    caught = 0
    for _ in range(40):
        bad = c.copy()
        pos = int(rng.integers(off + 160, off + 2000))
        bad[pos] ^= 1 << int(rng.integers(0, 8))
        try:
            y = oracle.decompress(bad)
            caught += int(not np.array_equal(y, x))  # undetected corruption must at least not crash
        except oracle.OracleError as e:
            assert e.name in ("CORRUPT_STREAM", "MALFORMED_BACKREF")
            caught += 1
    assert caught == 40


@pytest.mark.parametrize("group", [64, 128, 224])
@pytest.mark.parametrize("mode", ["byte", "bit"])
def test_wide_de_groups(group, mode):
    """Wide DE groups: the header carries de_group, verify_de checks the rule per de_group
    sequences, every de_group file is also a valid 32-group DE file (a wider group's start lies at or before
    the start of each of its 32-sequence groups), and the round trip holds."""
    x = datagen.wiki(150_000, seed=9)
    kw = dict(mode=mode, de=True, block_size=65536, de_group=group)
    if mode == "bit":
        kw.update(sub_block_seqs=0, sub_blocks_per_block=16)
    f = oracle.compress(x, **kw)
    assert f[10] == group
    assert oracle.verify_de(f) == 1
    g = f.copy()
    g[10] = 32
    assert oracle.verify_de(g) == 1
    assert np.array_equal(oracle.decompress(f), np.frombuffer(x, np.uint8) if isinstance(x, bytes) else x)
    f32 = oracle.compress(x, **dict(kw, de_group=32))
    assert len(f) >= len(f32) * 0.95   # wider groups only restrict the parse further (ratio cost reported)
