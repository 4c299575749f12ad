"""GPU compressor parity, `-m gpu`: gomp_compress_device must write the same file as the
oracle's compressor (oracle/oracle.c: greedy exhaustive longest match, package-merge, canonical codes) for the
same input and parameters, byte for byte -- the parse, the DE rule, the Huffman code lengths and the bit packing
are all pinned by that identity -- and the GPU decoder must restore the input from it."""
import numpy as np
import pytest
import torch

import datagen
import oracle
import paper_1606_00519_b200 as gomp

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _data(kind, n, seed=1):
    if kind == "zeros":
        return datagen.zeros(n)
    if kind.startswith("nested"):
        return datagen.nested(n, int(kind[6:]), seed=seed)
    return datagen.GENERATORS[kind](n, seed=seed)


def _gpu_compress(x, **kw):
    return gomp.compress_device(torch.from_numpy(np.ascontiguousarray(x)).to(DEV), **kw).cpu().numpy()


def _oracle_kw(kw):
    o = dict(kw)
    if o.get("mode") == "bit" and "sub_blocks_per_block" in o:
        o.setdefault("sub_block_seqs", 0)
    return o


@pytest.mark.parametrize("kind,n", [("wiki", 300_007), ("text", 200_000), ("matrix", 250_001), ("nested8", 150_000),
                                    ("random", 70_001), ("zeros", 90_000), ("text", 0), ("text", 1), ("text", 17)])
@pytest.mark.parametrize("mode", ["byte", "bit"])
@pytest.mark.parametrize("de", [True, False])
def test_gpu_compressor_matches_oracle(kind, n, mode, de):
    x = _data(kind, n)
    kw = dict(mode=mode, de=de, block_size=32768)
    if mode == "bit":
        kw.update(sub_blocks_per_block=16, sub_block_seqs=0)
    g = _gpu_compress(x, **kw)
    ref = oracle.compress(x, **_oracle_kw(kw))
    assert np.array_equal(g, ref), f"{g.size} vs {ref.size} bytes, first diff at {np.flatnonzero(g[:min(g.size, ref.size)] != ref[:min(g.size, ref.size)])[:1]}"
    if n:
        y = gomp.decompress(torch.from_numpy(g).to(DEV)).cpu().numpy()
        assert np.array_equal(y, x)


@pytest.mark.parametrize("cfg", [
    dict(block_size=16), dict(block_size=4096, window_size=1), dict(block_size=1 << 20),
    dict(block_size=65536, min_match=3, max_match=65), dict(block_size=65536, min_match=3, max_match=3),
    dict(block_size=65536, window_size=32768), dict(block_size=262144, de_group=128),
    dict(block_size=262144, sub_block_seqs=16), dict(block_size=131072, sub_blocks_per_block=300, sub_block_seqs=0),
    dict(block_size=65536, cwl=9), dict(block_size=65536, cwl=15),
])
@pytest.mark.parametrize("mode", ["byte", "bit"])
def test_gpu_compressor_parameters(cfg, mode):
    x = _data("wiki", 600_001, seed=7)
    kw = dict(mode=mode, de=True, **cfg)
    if mode == "byte":
        for k in ("sub_block_seqs", "sub_blocks_per_block", "cwl"):
            kw.pop(k, None)
    g = _gpu_compress(x, **kw)
    assert np.array_equal(g, gomp.compress(x, **kw).numpy())


def test_gpu_compressor_c2_size():
    """BASELINE C2 shape (256 KiB blocks, 16 sub-blocks/block, DE) on 64 MiB: identical to the host compressor."""
    x = datagen.wiki(64 << 20, seed=2)
    kw = dict(mode="bit", de=True, block_size=262144, sub_blocks_per_block=16)
    g = _gpu_compress(x, **kw)
    assert np.array_equal(g, gomp.compress(x, **kw).numpy())


def test_gpu_compressor_rejects_approximate_finders():
    x = torch.zeros(1000, dtype=torch.uint8, device=DEV)
    for kw in (dict(match_finder=1), dict(max_chain=8)):
        with pytest.raises(gomp.GompError):
            gomp.compress_device(x, mode="byte", **kw)


def test_gpu_compressor_argument_errors():
    """C-ABI error paths of gomp_compress_device: workspace too small, destination too small, misaligned
    buffers, bad parameters -- reported as statuses, nothing written out of bounds."""
    import ctypes
    x = torch.from_numpy(np.ascontiguousarray(datagen.wiki(200_000, seed=3))).to(DEV)
    p = gomp.params(mode="bit", sub_blocks_per_block=16)
    L = gomp.lib()
    need = ctypes.c_size_t(0)
    assert L.gomp_compress_device_workspace_size(x.numel(), ctypes.byref(p), ctypes.byref(need)) == 0
    cap = L.gomp_compress_bound(x.numel(), ctypes.byref(p))
    out = torch.empty(cap + 16, dtype=torch.uint8, device=DEV)
    ws = torch.empty(need.value + 16, dtype=torch.uint8, device=DEV)
    n = ctypes.c_size_t(0)
    s0 = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def call(dst, dcap, w, wn, pp=p):
        return L.gomp_compress_device(x.data_ptr(), x.numel(), dst, dcap, ctypes.byref(n), w, wn, ctypes.byref(pp), s0)

    assert call(out.data_ptr(), cap, ws.data_ptr(), need.value - 16) == -10          # WORKSPACE_TOO_SMALL
    assert call(out.data_ptr(), 1000, ws.data_ptr(), need.value) == -9               # DST_TOO_SMALL
    assert call(out.data_ptr() + 1, cap, ws.data_ptr(), need.value) == -1            # misaligned destination
    bad = gomp.params(mode="bit", sub_blocks_per_block=16)
    bad.de_group = 48
    assert call(out.data_ptr(), cap, ws.data_ptr(), need.value, bad) == -1           # invalid parameters
    assert call(out.data_ptr(), cap, ws.data_ptr(), need.value) == 0
    ref = gomp.compress(x.cpu().numpy(), p=p).numpy()
    assert n.value == ref.size and np.array_equal(out[: n.value].cpu().numpy(), ref)
