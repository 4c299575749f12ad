"""Host-side tests of libgompresso.so (CPU only): the C ABI loads and exports every symbol include/gomp.h
declares; the host compressor writes files the oracle decodes (and, with the exhaustive match finder, the very
same bytes as the oracle's compressor); header/table validation; the multi-GPU shard planner."""
import os
import re
import subprocess

import numpy as np
import pytest
import torch

import datagen
import oracle
import paper_1606_00519_b200 as gomp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "gomp.h")).read()
    return sorted(set(re.findall(r"\b(gomp_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", gomp.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (gomp_\w+)", out))
    declared = _declared()
    assert declared and set(declared) <= exported, set(declared) - exported
    assert set(declared) == set(gomp.EXPORTS)
    gomp.lib()  # loads
    assert gomp.lib().gomp_version() == 1


def test_library_not_named_libgomp():
    assert os.path.basename(gomp.LIB_PATH) == "libgompresso.so"


def test_status_strings():
    for code, name in gomp.STATUS.items():
        assert gomp.lib().gomp_status_string(code).decode() == name


@pytest.mark.parametrize("kind,n", [("wiki", 120_000), ("matrix", 90_000), ("random", 30_000), ("zeros", 40_000),
                                    ("nested4", 50_000), ("text", 0), ("text", 1), ("text", 17)])
@pytest.mark.parametrize("mode", ["byte", "bit"])
@pytest.mark.parametrize("de", [True, False])
def test_compressor_matches_oracle_bytes(kind, n, mode, de):
    if kind == "zeros":
        x = datagen.zeros(n)
    elif kind.startswith("nested"):
        x = datagen.nested(n, int(kind[6:]))
    else:
        x = datagen.GENERATORS[kind](n, seed=4)
    kw = dict(mode=mode, de=de, block_size=32768)
    if mode == "bit":
        kw.update(sub_block_seqs=0, sub_blocks_per_block=16)
    c = gomp.compress(x, **kw).numpy()
    ref = oracle.compress(x, **kw)
    assert np.array_equal(c, ref)


@pytest.mark.parametrize("group", [64, 128])
@pytest.mark.parametrize("mode", ["byte", "bit"])
def test_compressor_wide_de_groups_match_oracle(group, mode):
    x = datagen.wiki(200_000, seed=6)
    kw = dict(mode=mode, de=True, block_size=65536, de_group=group)
    if mode == "bit":
        kw.update(sub_block_seqs=0, sub_blocks_per_block=16)
    c = gomp.compress(x, **kw).numpy()
    assert np.array_equal(c, oracle.compress(x, **kw))
    assert gomp.get_info(c).de_group == group
    for bad in (0, 16, 48, 256):
        with pytest.raises(gomp.GompError):
            gomp.compress(x[:1000], **dict(kw, de_group=bad))


@pytest.mark.parametrize("threads", [1, 3, 8])
def test_compressor_deterministic_across_threads(threads):
    x = datagen.wiki(400_000, seed=9)
    a = gomp.compress(x, mode="bit", block_size=65536, n_threads=threads).numpy()
    b = gomp.compress(x, mode="bit", block_size=65536, n_threads=1).numpy()
    assert np.array_equal(a, b)
    assert np.array_equal(oracle.decompress(a), x)


@pytest.mark.parametrize("finder,chain", [(1, 0), (0, 4)])
def test_fast_match_finders_round_trip(finder, chain):
    x = datagen.wiki(300_000, seed=2)
    for mode in ("byte", "bit"):
        c = gomp.compress(x, mode=mode, de=True, block_size=65536, match_finder=finder, max_chain=chain).numpy()
        assert np.array_equal(oracle.decompress(c), x)
        assert oracle.verify_de(c)


def test_params_defaults_are_the_papers():
    p = gomp.params()
    assert (p.block_size, p.window_size, p.max_match, p.sub_block_seqs, p.cwl, p.min_staleness) == \
        (262144, 8192, 64, 16, 10, 1024)


def test_get_info_and_validation():
    x = datagen.text(50_000)
    c = gomp.compress(x, mode="bit", block_size=16384, sub_blocks_per_block=4)
    info = gomp.get_info(c)
    assert info.uncompressed_len == 50_000 and info.n_blocks == 4 and info.mode == 1 and info.de == 1
    assert info.file_len == c.numel() and info.n_sub_total == 16
    gomp.validate_tables(c)
    bad = c.clone()
    bad[0] = 0
    with pytest.raises(gomp.GompError) as e:
        gomp.get_info(bad)
    assert e.value.name == "BAD_MAGIC"
    bad = c.clone()
    bad[4] = 9
    with pytest.raises(gomp.GompError) as e:
        gomp.get_info(bad)
    assert e.value.name == "UNSUPPORTED_VERSION"
    with pytest.raises(gomp.GompError) as e:
        gomp.get_info(c[:63])
    assert e.value.name == "TRUNCATED"
    bad = c.clone()
    bad[64 + 32 + 12] += 1  # n_seq of block 1 -> n_sub mismatch
    with pytest.raises(gomp.GompError) as e:
        gomp.validate_tables(bad)
    assert e.value.name == "HEADER_INCONSISTENT" and e.value.block == 1


def test_workspace_size():
    x = datagen.text(70_000)
    cb = gomp.compress(x, mode="byte", block_size=16384)
    assert gomp.workspace_size(gomp.get_info(cb)) == 1024
    ct = gomp.compress(x, mode="bit", block_size=16384)
    info = gomp.get_info(ct)
    assert gomp.workspace_size(info) >= 1024 + info.n_blocks * info.max_block_tokens


@pytest.mark.parametrize("n_dev", [1, 2, 3, 4, 8])
def test_plan_shards_balanced(n_dev):
    import struct
    x = datagen.wiki(2_000_000, seed=3)
    c = gomp.compress(x, mode="bit", block_size=65536).numpy()
    first = gomp.plan_shards(c, n_dev)
    nb = gomp.get_info(c).n_blocks
    assert first[0] == 0 and first[-1] == nb and all(a <= b for a, b in zip(first, first[1:]))
    sizes = [sum(struct.unpack_from("<I", c.tobytes(), 64 + 32 * b + 8)[0] for b in range(first[d], first[d + 1]))
             for d in range(n_dev)]
    avg_block = sum(sizes) / nb
    assert max(sizes) - min(sizes) <= 2 * avg_block + 1


def test_decoder_choice_follows_the_measured_crossover():
    """huff_variant mirrors the launcher: the speculative warp decoder from a mean of 8192 bits per sub-block
    (profiles/r01_ncu_summary.md crossover), the thread-per-sub-block decoder below."""
    x = datagen.matrix(400_000, seed=2)
    for k, want in ((4, "warp"), (64, "thread")):
        c = gomp.compress(x, mode="bit", de=True, block_size=131072, sub_blocks_per_block=k, sub_block_seqs=0)
        info = gomp.get_info(c)
        avg = (info.file_len - info.payload_base) * 8 / info.n_sub_total
        assert gomp.huff_variant(info) == ("warp" if avg >= 8192 else "thread") == want, avg


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    """No CPU fallback: without libgompresso.so every entry point raises instead of computing on the host."""
    monkeypatch.setattr(gomp, "LIB_PATH", str(tmp_path / "libgompresso.so"))
    monkeypatch.setattr(gomp, "_lib", None)
    x = np.frombuffer(b"abcabcabcabc" * 100, dtype=np.uint8)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        gomp.compress(x)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        gomp.get_info(np.zeros(64, dtype=np.uint8))


def test_decompress_rejects_host_tensors():
    """The decompression entry points take CUDA tensors only (no silent host path)."""
    c = gomp.compress(np.frombuffer(b"hello hello hello" * 50, dtype=np.uint8))
    info = gomp.get_info(c)
    t = torch.zeros(16, dtype=torch.uint8)
    with pytest.raises(ValueError, match="no CPU fallback"):
        gomp.decompress_into(info, c, t, t)


@pytest.mark.parametrize("mode", ["byte", "bit"])
@pytest.mark.parametrize("kind,n", [("wiki", 700_001), ("matrix", 300_000)])
def test_shard_file_rebased(mode, kind, n):
    """gomp_shard_file: a shard of blocks [b0, b1) is a valid standalone file (host table
    validation) that the oracle decodes to bytes [b0 * block_size, ...) of the input; its size is O(shard)."""
    x = datagen.GENERATORS[kind](n, seed=8)
    kw = dict(mode=mode, de=True, block_size=32768)
    if mode == "bit":
        kw.update(sub_block_seqs=0, sub_blocks_per_block=8)
    c = gomp.compress(x, **kw)
    info = gomp.get_info(c)
    for b0, b1 in [(0, info.n_blocks), (0, 1), (3, 7), (info.n_blocks - 2, info.n_blocks), (5, 5)]:
        s = gomp.shard_file(c, b0, b1 - b0)
        gomp.validate_tables(s)
        si = gomp.get_info(s)
        assert si.n_blocks == b1 - b0
        y = oracle.decompress(s.numpy()) if b1 > b0 else np.zeros(0, np.uint8)
        lo = b0 * info.block_size
        assert np.array_equal(y, x[lo: lo + si.uncompressed_len])
        assert len(y) == min(b1 * info.block_size, n) - min(lo, n)
        if b1 - b0 == 1:
            assert si.file_len < info.file_len / 4
    with pytest.raises(gomp.GompError):
        gomp.shard_file(c, info.n_blocks - 1, 2)
