"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle, byte for byte (`-m gpu`).

Inputs are seeded synthetic data of the paper's workloads. Files come from the host compressor
(never from the CUDA path); expected bytes come from oracle.decompress() (and equal the original input).
Sizes span several blocks and warp groups with ragged tails; the full BASELINE.json sizes are covered by
test_full_size_* (all bytes vs the input; oracle on sampled blocks).
"""
import numpy as np
import pytest
import torch

import datagen
import oracle
import paper_1606_00519_b200 as gomp
from fmt_util import byte_file

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _data(kind, n, seed=1):
    if kind == "zeros":
        return datagen.zeros(n)
    if kind.startswith("nested"):
        return datagen.nested(n, int(kind[6:]), seed=seed)
    return datagen.GENERATORS[kind](n, seed=seed)


def _gpu(c, strategy="auto", **kw):
    return gomp.decompress(torch.as_tensor(np.asarray(c)).to(DEV), strategy=strategy, **kw)


def _check(c, x, strategies, **kw):
    ref = oracle.decompress(np.asarray(c))
    assert np.array_equal(ref, x)
    for s in strategies:
        y = _gpu(c, s, **kw).cpu().numpy()
        assert y.shape == ref.shape
        if not np.array_equal(y, ref):
            bad = np.flatnonzero(y != ref)
            raise AssertionError(f"strategy {s}: {bad.size} bytes differ, first at {bad[0]}")


KINDS = [("wiki", 1_100_003), ("text", 1 << 20), ("matrix", 700_001), ("nested8", 300_000), ("nested32", 200_000),
         ("random", 150_001), ("zeros", 100_000)]


@pytest.mark.parametrize("kind,n", KINDS)
@pytest.mark.parametrize("de", [True, False])
def test_byte_parity(kind, n, de):
    x = _data(kind, n)
    c = gomp.compress(x, mode="byte", de=de, block_size=65536)
    _check(c, x, ["de", "mrr", "sc"] if de else ["mrr", "sc", "de"])


@pytest.mark.parametrize("kind,n", KINDS)
@pytest.mark.parametrize("de", [True, False])
@pytest.mark.parametrize("sub", [("k", 16), ("S", 16)])
def test_bit_parity(kind, n, de, sub):
    x = _data(kind, n)
    kw = dict(sub_blocks_per_block=sub[1], sub_block_seqs=0) if sub[0] == "k" else dict(sub_block_seqs=sub[1])
    c = gomp.compress(x, mode="bit", de=de, block_size=65536, **kw)
    _check(c, x, ["auto", "mrr"] if de else ["auto", "sc"])


@pytest.mark.parametrize("group", [64, 128, 224])
@pytest.mark.parametrize("kind,n", [("wiki", 1_100_003), ("nested8", 300_000), ("matrix", 500_001)])
@pytest.mark.parametrize("mode", ["byte", "bit"])
def test_wide_de_group_parity(group, kind, n, mode):
    """Wide DE groups: the batch LZ77 kernel needs no wait inside a 128-sequence batch."""
    x = _data(kind, n)
    kw = dict(sub_blocks_per_block=16, sub_block_seqs=0) if mode == "bit" else {}
    c = gomp.compress(x, mode=mode, de=True, block_size=65536, de_group=group, **kw)
    _check(c, x, ["auto", "mrr"])
    _, st = _gpu(c, "de", return_stats=True)
    assert st["de_fallback_groups"] == 0


@pytest.mark.parametrize("cfg", [
    dict(block_size=16), dict(block_size=4096, window_size=1), dict(block_size=1 << 20),
    dict(block_size=32768, min_match=3, max_match=65), dict(block_size=32768, min_match=3, max_match=3),
    dict(block_size=32768, window_size=32768), dict(block_size=262144, sub_blocks_per_block=1, sub_block_seqs=0),
    dict(block_size=262144, sub_block_seqs=1), dict(block_size=262144, sub_blocks_per_block=300, sub_block_seqs=0),
])
@pytest.mark.parametrize("mode", ["byte", "bit"])
def test_parameter_edges(cfg, mode):
    x = datagen.wiki(600_000, seed=5)
    kw = dict(cfg)
    if mode == "bit" and "sub_block_seqs" not in kw:
        kw["sub_block_seqs"] = 16
    if mode == "byte":
        kw.pop("sub_block_seqs", None)
        kw.pop("sub_blocks_per_block", None)
    c = gomp.compress(x, mode=mode, **kw)
    _check(c, x, ["auto", "mrr"])


@pytest.mark.parametrize("cwl", [9, 11, 12, 15])
def test_code_length_limits(cwl):
    """cwl > 11 exercises the canonical path for codes longer than the shared-memory table index."""
    x = datagen.matrix(500_000, seed=8)
    c = gomp.compress(x, mode="bit", cwl=cwl, block_size=131072, sub_block_seqs=0, sub_blocks_per_block=8)
    _check(c, x, ["auto"])


@pytest.mark.parametrize("cwl", [10, 15])
@pytest.mark.parametrize("kind", ["wiki", "random"])
def test_split_grid_decode(cwl, kind):
    """A few blocks with 32 long sub-blocks each take the split speculative-decoder grid (two CTAs per block,
    half of its sub-blocks each), with table-index and longer (canonical path) codes."""
    x = (datagen.wiki if kind == "wiki" else datagen.random_bytes)(3 * 262144 - 4099, seed=31)
    c = gomp.compress(x, mode="bit", cwl=cwl, block_size=262144, sub_block_seqs=0, sub_blocks_per_block=32)
    assert gomp.huff_variant(gomp.get_info(c)) == "warp"
    _check(c, x, ["auto"])


@pytest.mark.parametrize("n", [0, 1, 15, 16, 17, 65535, 65536, 65537, 3 * 65536 - 1])
@pytest.mark.parametrize("mode", ["byte", "bit"])
def test_sizes_and_ragged_tails(n, mode):
    x = datagen.text(n, seed=12)
    c = gomp.compress(x, mode=mode, block_size=65536, sub_block_seqs=16)
    ref = oracle.decompress(c.numpy())
    y = _gpu(c).cpu().numpy()
    assert np.array_equal(y, ref) and np.array_equal(ref, x)


def test_hand_built_mrr_chain():
    """Adversarial chain: lane i reads lane i-1's back-reference output (3 MRR rounds)."""
    seqs = [(8, 8, 8), (0, 8, 8), (0, 8, 8)]
    f = byte_file([(seqs, b"ABCDEFGH")], block_size=64)
    for s in ("mrr", "sc", "de"):
        y, st = _gpu(f, s, return_stats=True)
        assert bytes(y.cpu().numpy()) == b"ABCDEFGH" * 4
    y, st = _gpu(f, "mrr", return_stats=True)
    assert st["rounds"][3] == 1 and st["bytes"][1:4] == [8, 8, 8]
    _, st = _gpu(f, "de", return_stats=True)
    assert st["de_fallback_groups"] == 1


@pytest.mark.parametrize("kind", ["wiki", "matrix", "nested4", "nested16", "nested32"])
@pytest.mark.parametrize("mode", ["byte", "bit"])
def test_mrr_statistics_match_oracle_model(kind, mode):
    x = _data(kind, 400_000, seed=3)
    c = gomp.compress(x, mode=mode, de=False, block_size=65536, sub_block_seqs=16)
    hist, nbytes = oracle.mrr_simulate(c.numpy())
    y, st = _gpu(c, "mrr", return_stats=True)
    assert np.array_equal(y.cpu().numpy(), x)
    assert st["rounds"] == [int(v) for v in hist]
    assert st["bytes"][1:] == [int(v) for v in nbytes[1:]]
    cd = gomp.compress(x, mode=mode, de=True, block_size=65536, sub_block_seqs=16)
    hd, bd = oracle.mrr_simulate(cd.numpy())
    for s in ("de", "mrr"):
        y, st = _gpu(cd, s, return_stats=True)
        assert np.array_equal(y.cpu().numpy(), x)
        assert st["rounds"] == [int(v) for v in hd] and st["de_fallback_groups"] == 0


def _expect(status, f, strategy="auto"):
    with pytest.raises(gomp.GompError) as e:
        _gpu(f, strategy)
    assert e.value.name == status, e.value


def test_device_errors_byte():
    _expect("MALFORMED_BACKREF", byte_file([([(4, 4, 2)], b"abcd")], block_size=16))          # overlap (R2)
    _expect("MALFORMED_BACKREF", byte_file([([(2, 4, 5)], b"ab")], block_size=16))            # before block
    f = byte_file([([(65, 65, 65)], b"a" * 65)], block_size=144, max_match=64)                # L > max_match
    _expect("MALFORMED_BACKREF", f)
    with pytest.raises(oracle.OracleError) as e:
        oracle.decompress(f)
    assert e.value.name == "MALFORMED_BACKREF"
    _expect("MALFORMED_BACKREF", byte_file([([(16, 0, 0)], b"a" * 16), ([(8, 4, 8), (0, 4, 12)], b"b" * 8)],
                                           block_size=16, window=8))                          # beyond window
    f = byte_file([([(3, 0, 0)], b"abc")], block_size=16)
    f[24] = 4
    _expect("CORRUPT_STREAM", f)
    x = datagen.text(100_000)
    c = gomp.compress(x, mode="byte", block_size=16384).numpy().copy()
    c[64 + 32 * 2 + 12] += 1     # n_seq of block 2: payload no longer adds up
    with pytest.raises(gomp.GompError) as e:
        _gpu(c)
    assert e.value.name in ("CORRUPT_STREAM", "MALFORMED_BACKREF", "HEADER_INCONSISTENT") and e.value.block == 2


# Corrupted files: the GPU must raise iff the oracle raises (the definition: sequential expansion, P:767-779,
# with the FORMAT.md §2 checks), and when both succeed the outputs must be identical byte for byte. Which status
# wins may differ (the oracle stops at the first bad sequence of the first bad block, the device reports the
# first error any CTA records), so only the class is compared: every device status is a format error.
FORMAT_ERRORS = ("CORRUPT_STREAM", "MALFORMED_BACKREF", "HEADER_INCONSISTENT")


def _agree(f, strategies=("auto",), huff=None):
    """Run f through the oracle and the GPU (each strategy); returns (oracle status or 'ok', gpu statuses)."""
    try:
        ref, o_st = oracle.decompress(f), "ok"
    except oracle.OracleError as e:
        ref, o_st = None, e.name
    g_sts = []
    for s in strategies:
        try:
            y, g_st = _gpu(f, s, huff=huff).cpu().numpy(), "ok"
        except gomp.GompError as e:
            y, g_st = None, e.name
        assert (o_st == "ok") == (g_st == "ok"), f"strategy {s}: oracle {o_st}, gpu {g_st}"
        if g_st == "ok":
            assert np.array_equal(y, ref), f"strategy {s}: both accept, outputs differ"
        else:
            assert g_st in FORMAT_ERRORS, g_st
        g_sts.append(g_st)
    return o_st, g_sts


def _flip(c, rng, lo, hi, n):
    bad = c.copy()
    for _ in range(n):
        pos = int(rng.integers(lo, hi))
        bad[pos] ^= np.uint8(1 << int(rng.integers(0, 8)))
    return bad


@pytest.mark.parametrize("sub,huff", [(("k", 8), None), (("S", 16), None), (("k", 8), "thread")])
def test_device_errors_bit_fuzz(sub, huff):
    """Bit flips in Bit payloads (trees, bitstreams), block-table and sub-table entries: GPU raises iff the
    oracle does, identical output otherwise. k=8 sub-blocks of ~3 kbit per block go through the speculative
    warp decoder, S=16 through the thread decoder with staged rounds, k=8 forced onto the thread decoder through
    its one-warp CTAs that stage nothing (register window)."""
    import struct
    x = datagen.wiki(200_000, seed=2)
    kw = dict(sub_block_seqs=0, sub_blocks_per_block=sub[1]) if sub[0] == "k" else dict(sub_block_seqs=sub[1])
    c = gomp.compress(x, mode="bit", block_size=32768, **kw).numpy()
    info = gomp.get_info(c)
    off = struct.unpack_from("<Q", c.tobytes(), 64)[0]
    rng = np.random.default_rng(0)
    seen = {}
    regions = [(off, off + 3000), (off, len(c) - 16), (64, 64 + 32 * info.n_blocks), (64 + 32 * info.n_blocks, off)]
    for i in range(80):
        lo, hi = regions[i % len(regions)]
        o_st, g = _agree(_flip(c, rng, lo, hi, int(rng.integers(1, 3))), ("auto", "mrr"), huff=huff)
        seen[o_st] = seen.get(o_st, 0) + 1
    assert seen.get("CORRUPT_STREAM", 0) > 0, seen
    bad = c.copy()
    bad[64 + 12] += 1  # n_seq of block 0
    with pytest.raises(gomp.GompError) as e:
        _gpu(bad)
    assert e.value.name in ("HEADER_INCONSISTENT", "CORRUPT_STREAM") and e.value.block == 0
    with pytest.raises(oracle.OracleError):
        oracle.decompress(bad)
    bad = c.copy()
    bad[64 + 28] += 1  # n_sub of block 0: no longer ceil(n_seq / S)
    with pytest.raises(gomp.GompError) as e:
        _gpu(bad)
    assert e.value.name == "HEADER_INCONSISTENT" and e.value.block == 0
    with pytest.raises(oracle.OracleError):
        oracle.decompress(bad)
    assert np.array_equal(_gpu(c).cpu().numpy(), x)


@pytest.mark.parametrize("de", [True, False])
@pytest.mark.parametrize("n,bs", [(300_000, 16384), (2_200_000, 4096)])
def test_device_errors_byte_fuzz(de, n, bs):
    """Byte flips in Byte-format records and literals (the LZ77 kernels read them straight from the file) and in
    the block table: GPU raises iff the oracle does, for every strategy, identical output otherwise. 537 blocks of
    4 KiB take the throughput LZ77 copy variant, 19 blocks of 16 KiB the latency variant."""
    import struct
    x = datagen.wiki(n, seed=21)
    c = gomp.compress(x, mode="byte", de=de, block_size=bs).numpy()
    nb = gomp.get_info(c).n_blocks
    off = struct.unpack_from("<Q", c.tobytes(), 64)[0]
    rng = np.random.default_rng(7)
    seen = {}
    for i in range(60):
        lo, hi = (off, len(c) - 16) if i % 4 else (64, 64 + 32 * nb)
        o_st, g = _agree(_flip(c, rng, lo, hi, int(rng.integers(1, 4))), ("auto", "de", "mrr", "sc"))
        seen[o_st] = seen.get(o_st, 0) + 1
    assert set(seen) & {"CORRUPT_STREAM", "MALFORMED_BACKREF"}, seen   # record damage is detected
    assert np.array_equal(_gpu(c).cpu().numpy(), x)                      # and the device is still fine


def test_device_errors_byte_record_fields():
    """Every field of a Byte record pushed just past its FORMAT.md §2 limit, one at a time, in the first and in a
    later warp group of a block: the oracle and the GPU (all strategies) both reject, and both accept the limit."""
    seqs = [(5, 4, 5)] + [(1, 4, 5)] * 40
    lits = bytes(range(65, 70)) + bytes(40)
    good = [(seqs, lits)]
    for blocks in (good, [([(256, 0, 0)], b"x" * 256)] + good):
        f = byte_file(blocks, block_size=256)
        assert _agree(f, ("auto", "de", "mrr", "sc"))[0] == "ok"
    cases = {
        "L > max_match (65 > 64)": ([(65, 0, 0), (0, 65, 65)], b"q" * 65, dict(max_match=64)),
        "L > max_match, min_match 3": ([(70, 0, 0), (0, 64, 64)], b"q" * 70, dict(min_match=3, max_match=63)),
        "dist < L (overlap, R2)": ([(4, 0, 0), (0, 5, 4)], b"abcd", {}),
        "dist > window (R9)": ([(64, 0, 0), (0, 8, 33)], b"w" * 64, dict(window=32)),
        "dist > dst (before the block)": ([(4, 0, 0), (0, 4, None)], b"abcd", {}),
    }
    for name, (sq, lt, kw) in cases.items():
        for pad in (0, 40):       # first group, or a later group of the same block
            # None: dist = dst + 1 (the source starts one byte before the block)
            sq2 = [(a, b, d if d is not None else pad + 5) for a, b, d in sq]
            s2 = [(1, 0, 0)] * pad + sq2
            l2 = b"p" * pad + lt
            total = sum(a + b for a, b, _ in s2)
            f = byte_file([(s2, l2)], block_size=max(16, (total + 15) // 16 * 16), **kw)
            o_st, g = _agree(f, ("auto", "de", "mrr", "sc"))
            assert o_st == "MALFORMED_BACKREF" and set(g) == {"MALFORMED_BACKREF"}, (name, pad, o_st, g)
    # empty records (lit_len 0, no back-reference) are valid sequences for the definition, also past ulen
    f = byte_file([([(3, 0, 0)] + [(0, 0, 0)] * 40 + [(1, 4, 4)], b"abcd")], block_size=16)
    assert _agree(f, ("auto", "de", "mrr", "sc"))[0] == "ok"


def test_blocks_range_and_shards():
    """gomp_decompress_blocks on shard ranges == the matching slice of the whole output."""
    x = datagen.wiki(3_000_000, seed=6)
    c = gomp.compress(x, mode="bit", block_size=131072)
    info = gomp.get_info(c)
    d = c.to(DEV)
    for n_dev in (2, 3, 8):
        first = gomp.plan_shards(c, n_dev)
        parts = []
        for k in range(n_dev):
            b0, b1 = first[k], first[k + 1]
            lo, hi = b0 * info.block_size, min(b1 * info.block_size, info.uncompressed_len)
            out = torch.empty(max(hi - lo, 1), dtype=torch.uint8, device=DEV)
            ws = torch.empty(gomp.workspace_size(info, max(b1 - b0, 1)), dtype=torch.uint8, device=DEV)
            gomp.decompress_into(info, d, out, ws, first_block=b0, n_blocks=b1 - b0)
            e = gomp.read_error(ws)
            assert e.status == 0
            parts.append(out[: hi - lo].cpu().numpy())
        assert np.array_equal(np.concatenate(parts), x)


@pytest.mark.parametrize("mode", ["byte", "bit"])
def test_lz77_copy_variants(mode):
    """The DE LZ77 kernel has three variants chosen by grid size: 4-warp batches with the
    instruction-lean copies (full grids), 4-warp batches with the load-first copies (<= 3 CTAs per SM) and 16-warp
    batches (<= 1 CTA per SM). The same 600-block file decoded whole, in 300-block ranges and in 64-block ranges
    must equal the input and the oracle."""
    x = datagen.wiki(600 * 65536 - 777, seed=12)
    c = gomp.compress(x, mode=mode, de=True, block_size=65536, sub_blocks_per_block=8)
    info = gomp.get_info(c)
    assert info.n_blocks == 600
    assert np.array_equal(_gpu(c).cpu().numpy(), x)
    d = c.to(DEV)
    out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device=DEV)
    ws = torch.empty(gomp.workspace_size(info, 64), dtype=torch.uint8, device=DEV)
    ws = torch.empty(gomp.workspace_size(info, 300), dtype=torch.uint8, device=DEV)
    for rng in (300, 64):
        out.zero_()
        for b0 in range(0, 600, rng):
            nb = min(rng, 600 - b0)
            gomp.decompress_into(info, d, out[b0 * 65536:], ws, first_block=b0, n_blocks=nb)
            assert gomp.read_error(ws).status == 0
        y = out.cpu().numpy()
        assert np.array_equal(y, x), rng
    cn = c.numpy()
    for b in (0, 317, 599):
        ref = oracle.decompress_blocks(cn, b, b + 1, 65536)
        assert np.array_equal(y[b * 65536: b * 65536 + len(ref)], ref)


def test_host_end_to_end():
    x = datagen.wiki(2_000_000, seed=7)
    for mode in ("byte", "bit"):
        c = gomp.compress(x, mode=mode).pin_memory()
        y = gomp.decompress_host(c, device=DEV)
        assert np.array_equal(y.numpy(), x)


@pytest.mark.parametrize("mode", ["byte", "bit"])
@pytest.mark.parametrize("n,bs", [(700_001, 16384), (3_000_017, 8192), (100_000, 65536), (0, 65536)])
def test_host_pipeline(mode, n, bs):
    """gomp_decompress_host cuts the blocks into chunks of doubling size whose copies and kernels overlap on
    internal streams; output must equal the input, for every chunk count including one, in the "In/Out" mode
    and in the "In" mode (h_dst NULL: the output stays on the device)."""
    x = datagen.wiki(n, seed=17)
    c = gomp.compress(x, mode=mode, block_size=bs).pin_memory()
    for strategy in ("auto", "mrr"):
        y = gomp.decompress_host(c, device=DEV, strategy=strategy)
        assert np.array_equal(y.numpy(), x)
        z = gomp.decompress_host(c, device=DEV, strategy=strategy, in_mode=True)
        assert z.is_cuda and np.array_equal(z.cpu().numpy(), x)


def test_host_pipeline_reports_late_error():
    """A corrupt block in the last chunk of the pipelined host path is reported with its block index."""
    x = datagen.wiki(3_000_017, seed=18)
    c = gomp.compress(x, mode="byte", block_size=8192).numpy().copy()
    info = gomp.get_info(c)
    b = info.n_blocks - 3
    off = int(np.frombuffer(c[64 + 32 * b: 72 + 32 * b].tobytes(), dtype=np.uint64)[0])
    c[off: off + 64] = 0xff                       # first records of block b: lit_len 1023, bad fields
    with pytest.raises(gomp.GompError) as ei:
        gomp.decompress_host(torch.from_numpy(c).pin_memory(), device=DEV)
    assert ei.value.block == b


def test_bad_arguments():
    x = datagen.text(10_000)
    c = gomp.compress(x, mode="byte", block_size=4096)
    info = gomp.get_info(c)
    d = c.to(DEV)
    out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device=DEV)
    ws = torch.empty(gomp.workspace_size(info), dtype=torch.uint8, device=DEV)
    with pytest.raises(gomp.GompError) as e:
        gomp.decompress_into(info, d, out[: info.uncompressed_len - 1], ws)
    assert e.value.name == "DST_TOO_SMALL"
    with pytest.raises(gomp.GompError) as e:
        gomp.decompress_into(info, d[: info.file_len - 1], out, ws)
    assert e.value.name == "TRUNCATED"
    with pytest.raises(gomp.GompError) as e:
        gomp.decompress_into(info, d, out, ws, strategy=9)
    assert e.value.name == "INVALID_ARG"
    with pytest.raises(gomp.GompError) as e:
        gomp.decompress_into(info, d, out[1:], ws)
    assert e.value.name == "INVALID_ARG"  # misaligned output


@pytest.mark.slow
@pytest.mark.parametrize("cfg", ["C1", "C2", "C3-byte-mrr", "C3-byte-de", "C3-bit-de"])
def test_full_size_configs(cfg):
    """BASELINE.json configs at full size, in the launch configuration bench.py times: every output byte vs
    the original input, and the oracle on sampled blocks."""
    if cfg == "C1":
        x = datagen.text(1 << 20, seed=1)
        c = gomp.compress(x, mode="byte", de=True, block_size=65536)
    elif cfg == "C2":
        x = datagen.wiki(256 << 20, seed=2)
        c = gomp.compress(x, mode="bit", de=True, block_size=262144, sub_blocks_per_block=16)
    elif cfg == "C3-byte-mrr":
        x = datagen.nested(256 << 20, 8, seed=3)
        c = gomp.compress(x, mode="byte", de=False, block_size=262144)
    elif cfg == "C3-byte-de":
        x = datagen.nested(256 << 20, 8, seed=3)
        c = gomp.compress(x, mode="byte", de=True, block_size=262144)
    else:
        x = datagen.nested(256 << 20, 8, seed=3)
        c = gomp.compress(x, mode="bit", de=True, block_size=262144, sub_block_seqs=16)
    info = gomp.get_info(c)
    y = _gpu(c).cpu().numpy()
    assert np.array_equal(y, x)
    rng = np.random.default_rng(0)
    cn = c.numpy()
    bs = info.block_size
    for b in sorted(set([0, info.n_blocks - 1] + [int(v) for v in rng.integers(0, info.n_blocks, 6)])):
        ref = oracle.decompress_blocks(cn, b, b + 1, bs)
        assert np.array_equal(y[b * bs: b * bs + len(ref)], ref)


@pytest.mark.parametrize("kind", ["wiki", "matrix", "nested2", "nested32", "random", "zeros", "text"])
@pytest.mark.parametrize("k", [1, 4, 8, 16, 40, 64])
def test_warp_speculative_decode(kind, k):
    """Long sub-blocks (k per 256 KiB block) take the speculative decoder with groups of 8, 4, 2 or 1 warps (by
    the mean sub-block size: k = 1/4 -> 8, 8 -> 4, 16 -> 2, 40/64 -> 1 on text); incompressible data (1023-literal
    runs, R10) takes its serial fallback. Output must equal the oracle's bit for bit."""
    x = _data(kind, 1_500_007, seed=13)
    c = gomp.compress(x, mode="bit", de=kind != "nested2", block_size=262144, sub_block_seqs=0, sub_blocks_per_block=k)
    _check(c, x, ["auto"])


@pytest.mark.parametrize("kind", ["wiki", "matrix", "text", "nested8"])
@pytest.mark.parametrize("bs,k", [(65536, 16), (65536, 4), (131072, 24), (1 << 20, 16)])
def test_warp_speculative_short_chunks(kind, bs, k):
    """Sub-blocks whose 32 lane chunks hold fewer symbols than the self-sync window (kRec)."""
    x = _data(kind, 2_000_003, seed=21)
    c = gomp.compress(x, mode="bit", de=True, block_size=bs, sub_block_seqs=0, sub_blocks_per_block=k)
    _check(c, x, ["auto"])


@pytest.mark.parametrize("kind", ["wiki", "matrix", "nested8", "random", "zeros"])
@pytest.mark.parametrize("sub", [("k", 16), ("k", 3), ("S", 16), ("S", 200)])
@pytest.mark.parametrize("huff", ["thread", "warp"])
def test_forced_decoder_variant(kind, sub, huff):
    """Both Bit decoders (thread per sub-block, warp per sub-block) on every sub-block shape, whichever one the
    launcher would pick: same output as the oracle, bit for bit."""
    x = _data(kind, 700_001, seed=31)
    kw = dict(sub_blocks_per_block=sub[1], sub_block_seqs=0) if sub[0] == "k" else dict(sub_block_seqs=sub[1])
    c = gomp.compress(x, mode="bit", de=True, block_size=131072, **kw)
    _check(c, x, ["auto"], huff=huff)


def _heavy_data(n_units=54, seed=5, n_light=12):
    """Units of one 16-sequence stretch of ~100 random literals per sequence (a ~13 kbit sub-block) followed by
    n_light x 16 sequences of 64-byte matches of a periodic pattern (~150 bits each): a few sub-blocks per round
    far longer than the mean, as a DE file's first group of every block (C3), here 19 of 256 in one round."""
    rng = np.random.default_rng(seed)
    period = rng.integers(0, 256, 61, dtype=np.uint8)
    light = np.tile(period, n_light * 16 * 64 // 61 + 1)[:n_light * 16 * 64]
    parts = []
    for _ in range(n_units):
        first = None
        for _ in range(16):
            r = rng.integers(0, 256, 100, dtype=np.uint8)
            first = r if first is None else first
            parts += [r, first[:8]]
        parts.append(light)
    return np.concatenate(parts)


def _heavy_per_round(c):
    """Deferred sub-blocks per thread-decoder round, by the kernel's rule (bits >= kSpecMinBits = 3072 and >= 8 x
    the round's mean), with the launcher's round size for a grid of few blocks."""
    a = np.asarray(c)
    info = gomp.get_info(a)
    t = a[64:64 + 32 * info.n_blocks].view(np.uint32).reshape(-1, 8)
    sub = a[64 + 32 * info.n_blocks:64 + 32 * info.n_blocks + 8 * info.n_sub_total].view(np.uint32).reshape(-1, 2)
    avg_sub = -(-info.n_sub_total // info.n_blocks)
    nt = min(256, max(32, (avg_sub + 31) // 32 * 32))
    res = []
    for b in range(info.n_blocks):
        bits = sub[t[b, 5]:t[b, 5] + t[b, 7], 0].astype(np.int64)
        for r0 in range(0, len(bits), nt):
            rb = bits[r0:r0 + nt]
            res.append(int(((rb >= 3072) & (rb * len(rb) >= 8 * rb.sum())).sum()))
    return res


@pytest.mark.parametrize("de", [False, True])
def test_thread_decoder_heavy_sub_blocks(de):
    """Thread decoder rounds holding sub-blocks far longer than the mean: those are deferred and decoded by a whole
    warp (speculative decoder, one warp); more than kMaxHeavy = 16 in one round (non-DE file: 19) leaves the rest
    to their own thread. Same output as the oracle with either decoder; corrupted heavy sub-blocks are rejected
    exactly when the oracle rejects them."""
    x = _heavy_data()
    c = gomp.compress(x, mode="bit", de=de, block_size=262144, sub_block_seqs=16)
    per_round = _heavy_per_round(c)
    assert max(per_round) > (16 if not de else 0), per_round
    assert gomp.huff_variant(gomp.get_info(c)) == "thread"
    _check(c, x, ["auto", "mrr"] if de else ["mrr"])
    _check(c, x, ["auto"], huff="warp")
    # 4 bit flips inside the first heavy sub-block of block 0, 16 times (the oracle rejects 8 / 5 of them)
    import struct
    a = np.asarray(c).copy()
    info = gomp.get_info(a)
    off = struct.unpack_from("<Q", a.tobytes(), 64)[0]
    sub = a[64 + 32 * info.n_blocks:64 + 32 * info.n_blocks + 8 * info.n_sub_total].view(np.uint32).reshape(-1, 2)
    k = int(np.flatnonzero(sub[:, 0] >= 3072)[0])
    start = int(sub[:k, 0].astype(np.int64).sum())
    lo = off + 160 + start // 8  # the 160-byte code-length header (kTreeBytes, FORMAT.md §3) precedes the bits
    rng = np.random.default_rng(7)
    seen = {}
    for _ in range(16):
        o_st, _ = _agree(_flip(a, rng, lo, lo + int(sub[k, 0]) // 8, 4), ("auto",))
        seen[o_st] = seen.get(o_st, 0) + 1
    assert sum(v for st, v in seen.items() if st != "ok") > 0, seen


@pytest.mark.parametrize("mode", ["byte", "bit"])
@pytest.mark.parametrize("n_dev", [1, 2, 3])
def test_decompress_sharded(mode, n_dev):
    """The multi-GPU path of one process with every shard on cuda:0 (one GPU here): each shard
    gets only the tables and its own payload range; the shard outputs, concatenated, equal the oracle's."""
    x = _data("wiki", 1_300_007, seed=17)
    kw = dict(sub_blocks_per_block=16, sub_block_seqs=0) if mode == "bit" else {}
    c = gomp.compress(x, mode=mode, de=True, block_size=65536, **kw)
    parts = gomp.decompress_sharded(c, [DEV] * n_dev)
    assert [p[0] for p in parts] == gomp.plan_shards(c, n_dev)[:-1]
    y = np.concatenate([p[1].cpu().numpy() for p in parts])
    assert np.array_equal(y, oracle.decompress(c.numpy()))


def test_decompress_sharded_reports_device_errors():
    """A corrupted payload in one shard's range is reported as a GompError naming that device."""
    x = _data("wiki", 600_001, seed=19)
    c = gomp.compress(x, mode="byte", de=True, block_size=65536).numpy().copy()
    info = gomp.get_info(c)
    first = gomp.plan_shards(c, 2)
    b = first[1]                                      # first block of the second shard
    e = c[64 + 32 * b: 64 + 32 * b + 32].view(np.uint32)
    off = int(e[0]) | (int(e[1]) << 32)
    c[off: off + 64] = 0xff                           # records with impossible back-references
    with pytest.raises(gomp.GompError):
        gomp.decompress_sharded(c, [DEV, DEV])


def _edge_source_block(rng, block_size, window=8192):
    """Sequences of one DE block whose back-reference sources end 0-3 bytes before their group's start: the word
    loads of the OR-assembled copies then also read bytes of the current group, which other lanes
    and warps are writing at that moment. Literal bytes are random, so a leaked neighbour byte shows."""
    seqs, lits, o = [], bytearray(), 0
    while True:
        og = o
        group = []
        for _ in range(32):
            lit = int(rng.integers(0, 7))
            L = int(rng.integers(4, 13))
            e = og - int(rng.integers(0, 4))                  # source end: at or just before the group start
            dst = o + lit
            if e - L < 0 or dst - (e - L) > window or o + lit + L > block_size - 64:
                L, d = 0, 0
            else:
                d = dst - (e - L)
            group.append((lit, L, d))
            lits += bytes(rng.integers(0, 256, lit, dtype=np.uint8))
            o += lit + L
        seqs += group
        if o > block_size - 1100:
            break
    while o < block_size:                                     # fill the block with literal-only sequences
        lit = min(1023, block_size - o)
        seqs.append((lit, 0, 0))
        lits += bytes(rng.integers(0, 256, lit, dtype=np.uint8))
        o += lit
    return seqs, bytes(lits)


@pytest.mark.parametrize("nblocks,bs", [(3, 16384), (40, 4096), (2, 65536), (200, 4096), (600, 4096)])
def test_or_copy_overread_bytes_discarded(nblocks, bs):
    """Directed test for the racecheck hazards of DESIGN.md §5: the OR-assembled word copies read up to 3 bytes on
    either side of a source range (the funnel-shift neighbours) and those bytes may be written concurrently by
    another lane or warp; they must never reach the output. Every source here ends 0-3 bytes before its group's
    start, so the over-read bytes are exactly the ones being written; run repeatedly, every strategy and copy
    variant (600 blocks of 4 KiB: 4-warp batches, throughput copies; 200 blocks: 4-warp batches, load-first
    copies; 2-40 blocks: 16-warp batches) must equal the sequential expansion byte for byte."""
    from fmt_util import expand
    rng = np.random.default_rng(bs + nblocks)
    blocks = [_edge_source_block(rng, bs) for _ in range(nblocks)]
    f = byte_file(blocks, block_size=bs, de=True)
    want = b"".join(expand(s, l) for s, l in blocks)
    ref = oracle.decompress(f)
    assert bytes(ref) == want
    assert oracle.verify_de(f)
    for s in ("de", "mrr", "sc"):
        for _ in range(5):
            y = _gpu(f, s).cpu().numpy()
            assert y.tobytes() == want, s


@pytest.mark.slow
@pytest.mark.parametrize("bs,sub", [(262144, "S16"), (1 << 20, 4), (65536, 16), (65536, 32)])
def test_c5_full_size(bs, sub):
    """C5 at its BASELINE size as bench_configs.py measures it: a 256 MiB MatrixMarket-shaped file's blocks tiled
    16x (4 GiB), one point per decoder (thread decoder with 16-sequence sub-blocks; speculative decoder with groups
    of 8 warps for 1 MiB / 4 sub-blocks, of 1 warp for 64 KiB / 16; the stage-less one-warp thread decoder for
    64 KiB / 32): every byte vs the input, sampled blocks vs the oracle."""
    import bench
    x = datagen.matrix(256 << 20, seed=5)
    kw = dict(sub_block_seqs=16) if sub == "S16" else dict(sub_block_seqs=0, sub_blocks_per_block=sub)
    c = gomp.compress(x, mode="bit", de=True, block_size=bs, **kw).numpy()
    nb, tiles = gomp.get_info(c).n_blocks, 16
    f = bench.tiled_shard(c, 0, nb * tiles)
    y = _gpu(f)
    xd = torch.from_numpy(x).to(DEV)
    n = len(x)
    assert y.numel() == n * tiles
    for t in range(tiles):
        assert torch.equal(y[t * n:(t + 1) * n], xd), t
    rng = np.random.default_rng(bs)
    for b in sorted(set([0, nb * tiles - 1] + [int(v) for v in rng.integers(0, nb * tiles, 4)])):
        ref = oracle.decompress_blocks(f, b, b + 1, bs)
        assert np.array_equal(y[b * bs:b * bs + len(ref)].cpu().numpy(), ref)


@pytest.mark.parametrize("world,tiles", [(8, 8), (3, 4)])
def test_bench_tiled_shards_full_size(world, tiles):
    """bench.py's multi-GPU data at full C2 size (one GPU here: the ranks' shards decoded one after another on
    cuda:0): the C2 file's blocks tiled `tiles` times, split by gomp_plan_shards, each rank's shard file
    (bench.tiled_shard) decoded by the CUDA path; every byte equals the tiled input and sampled blocks the
    oracle's decode of the shard."""
    import bench
    x = datagen.wiki(256 << 20, seed=2)
    c = gomp.compress(x, mode="bit", de=True, block_size=262144, sub_blocks_per_block=16).numpy()
    nb = gomp.get_info(c).n_blocks
    first = gomp.plan_shards(bench.tiled_tables(c, tiles), world)
    assert first[0] == 0 and first[-1] == nb * tiles
    xd = torch.from_numpy(x).to(DEV)
    bs = 262144
    rng = np.random.default_rng(world)
    for r in range(world):
        b0, b1 = first[r], first[r + 1]
        s = bench.tiled_shard(c, b0, b1)
        y = _gpu(s)
        assert y.numel() == (b1 - b0) * bs
        for t in range(b0 // nb, (b1 - 1) // nb + 1):                   # every byte: pieces of the tiled input
            j0, j1 = max(b0 - t * nb, 0), min(b1 - t * nb, nb)
            o = (t * nb + j0 - b0) * bs
            assert torch.equal(y[o:o + (j1 - j0) * bs], xd[j0 * bs:j1 * bs])
        for b in rng.integers(b0, b1, 2):
            ref = oracle.decompress_blocks(s, int(b) - b0, int(b) - b0 + 1, bs)
            assert np.array_equal(y[(int(b) - b0) * bs:(int(b) - b0 + 1) * bs].cpu().numpy(), ref)
