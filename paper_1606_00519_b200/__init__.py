"""paper_1606_00519_b200 — B200-native Gompresso decompression (arXiv 1606.00519).

Thin ctypes binding of libgompresso.so (include/gomp.h). Argument marshalling only: every step of the
decompression path runs in the library's sm_100a kernels; PyTorch supplies device memory and streams.
There is no CPU fallback — if the library or a CUDA device is missing, calls raise.

    c = compress(x, mode="bit", de=True)           # host CPU compressor -> torch.uint8 CPU tensor (a file)
    y = decompress(c.cuda())                        # CUDA tensor of the original bytes
"""
import ctypes
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgompresso.so")

MODES = {"byte": 0, "bit": 1}
STRATEGIES = {"auto": 0, "de": 1, "mrr": 2, "sc": 3}
FLAG_STATS = 0x100
FLAG_DECODE_ONLY = 0x200
FLAG_LZ77_ONLY = 0x400
FLAG_HUFF_THREAD = 0x800
FLAG_HUFF_WARP = 0x1000
STATUS = {0: "OK", -1: "INVALID_ARG", -2: "BAD_MAGIC", -3: "UNSUPPORTED_VERSION", -4: "TRUNCATED",
          -5: "HEADER_INCONSISTENT", -6: "CORRUPT_STREAM", -7: "MALFORMED_BACKREF", -8: "NO_PROGRESS",
          -9: "DST_TOO_SMALL", -10: "WORKSPACE_TOO_SMALL", -11: "CUDA", -12: "OOM"}


class GompError(RuntimeError):
    """A gomp_status != GOMP_OK; .status (int), .name, .block (device errors), .detail."""

    def __init__(self, status, block=0, detail=0, where=""):
        self.status = int(status)
        self.name = STATUS.get(self.status, str(status))
        self.block = int(block)
        self.detail = int(detail)
        super().__init__(f"{where}: {self.name} (block {self.block}, detail {self.detail:#x})")


class Params(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint32) for n in (
        "struct_size", "mode", "de", "block_size", "window_size", "min_match", "max_match", "sub_block_seqs",
        "sub_blocks_per_block", "cwl", "match_finder", "min_staleness", "max_chain", "n_threads", "de_group")]


class Info(ctypes.Structure):
    _fields_ = [("uncompressed_len", ctypes.c_uint64), ("file_len", ctypes.c_uint64),
                ("payload_base", ctypes.c_uint64), ("n_blocks", ctypes.c_uint32), ("n_sub_total", ctypes.c_uint32),
                ("max_block_tokens", ctypes.c_uint32)] + [(n, ctypes.c_uint32) for n in (
                    "mode", "de", "block_size", "window_size", "min_match", "max_match", "cwl", "version", "de_group")]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Error(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("block", ctypes.c_uint32), ("detail", ctypes.c_uint64)]


class Stats(ctypes.Structure):
    _fields_ = [("rounds", ctypes.c_uint64 * 33), ("bytes", ctypes.c_uint64 * 33),
                ("de_fallback_groups", ctypes.c_uint64)]


_lib = None
EXPORTS = ["gomp_version", "gomp_status_string", "gomp_params_default", "gomp_compress_bound", "gomp_compress",
           "gomp_get_info", "gomp_validate_tables", "gomp_decompress_workspace_size", "gomp_decompress",
           "gomp_decompress_blocks", "gomp_decompress_host", "gomp_decompress_error", "gomp_decompress_stats",
           "gomp_plan_shards", "gomp_compress_device_workspace_size", "gomp_compress_device", "gomp_shard_file"]


def lib():
    """Load libgompresso.so (raises if it is missing: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing: build it with `python __graft_entry__.py` (no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, sz, u32, u8p = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint32, ctypes.c_void_p
    L.gomp_version.restype = ctypes.c_int
    L.gomp_status_string.argtypes = [ctypes.c_int]
    L.gomp_status_string.restype = ctypes.c_char_p
    L.gomp_params_default.argtypes = [ctypes.POINTER(Params)]
    L.gomp_params_default.restype = None
    L.gomp_compress_bound.argtypes = [sz, ctypes.POINTER(Params)]
    L.gomp_compress_bound.restype = sz
    L.gomp_compress.argtypes = [u8p, sz, u8p, sz, ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(Params)]
    L.gomp_get_info.argtypes = [u8p, sz, ctypes.POINTER(Info)]
    L.gomp_validate_tables.argtypes = [u8p, sz, ctypes.POINTER(ctypes.c_uint32)]
    L.gomp_decompress_workspace_size.argtypes = [ctypes.POINTER(Info), u32, ctypes.POINTER(ctypes.c_size_t)]
    L.gomp_decompress.argtypes = [ctypes.POINTER(Info), u8p, sz, u8p, sz, vp, sz, ctypes.c_int, vp]
    L.gomp_decompress_blocks.argtypes = [ctypes.POINTER(Info), u32, u32, u8p, sz, u8p, sz, vp, sz, ctypes.c_int, vp]
    L.gomp_decompress_host.argtypes = [ctypes.POINTER(Info), u8p, sz, u8p, sz, u8p, u8p, vp, sz, ctypes.c_int, vp]
    L.gomp_compress_device_workspace_size.argtypes = [sz, ctypes.POINTER(Params), ctypes.POINTER(ctypes.c_size_t)]
    L.gomp_compress_device.argtypes = [u8p, sz, u8p, sz, ctypes.POINTER(ctypes.c_size_t), vp, sz,
                                       ctypes.POINTER(Params), vp]
    L.gomp_decompress_error.argtypes = [vp, vp, ctypes.POINTER(Error)]
    L.gomp_decompress_stats.argtypes = [vp, vp, ctypes.POINTER(Stats)]
    L.gomp_plan_shards.argtypes = [u8p, sz, ctypes.c_int, ctypes.POINTER(ctypes.c_uint32)]
    L.gomp_shard_file.argtypes = [u8p, sz, u32, u32, u8p, sz, ctypes.POINTER(ctypes.c_size_t)]
    for f in EXPORTS[2:]:
        if f not in ("gomp_params_default", "gomp_compress_bound"):
            getattr(L, f).restype = ctypes.c_int
    _lib = L
    return L


def _check(st, where):
    if st != 0:
        raise GompError(st, where=where)


def params(mode="bit", de=True, block_size=262144, window_size=8192, min_match=4, max_match=64,
           sub_block_seqs=None, sub_blocks_per_block=0, cwl=10, match_finder=0, min_staleness=1024, max_chain=0,
           n_threads=0, de_group=32):
    """gomp_params; defaults = the paper's setup. Passing sub_blocks_per_block (k) selects the
    "k sub-blocks per block" parametrisation (BASELINE config C2) unless sub_block_seqs is also given."""
    p = Params()
    lib().gomp_params_default(ctypes.byref(p))
    if sub_block_seqs is None:
        sub_block_seqs = 0 if sub_blocks_per_block else 16
    vals = dict(mode=MODES[mode] if isinstance(mode, str) else int(mode), de=int(bool(de)), block_size=block_size,
                window_size=window_size, min_match=min_match, max_match=max_match, sub_block_seqs=sub_block_seqs,
                sub_blocks_per_block=sub_blocks_per_block, cwl=cwl, match_finder=match_finder,
                min_staleness=min_staleness, max_chain=max_chain, n_threads=n_threads, de_group=de_group)
    for k, v in vals.items():
        setattr(p, k, int(v))
    return p


def _host_u8(x):
    if isinstance(x, torch.Tensor):
        if x.is_cuda:
            raise ValueError("compress() takes host data")
        return np.ascontiguousarray(x.numpy().view(np.uint8).reshape(-1))
    if isinstance(x, (bytes, bytearray, memoryview)):
        return np.frombuffer(bytes(x), dtype=np.uint8)
    return np.ascontiguousarray(np.asarray(x).view(np.uint8).reshape(-1))


def compress(x, p=None, **kw):
    """gomp_compress on the host CPU: returns the compressed file as a CPU torch.uint8 tensor."""
    src = _host_u8(x)
    p = p or params(**kw)
    cap = lib().gomp_compress_bound(len(src), ctypes.byref(p))
    if cap == 0:
        raise GompError(-1, where="gomp_compress_bound")
    out = np.empty(cap, dtype=np.uint8)
    n = ctypes.c_size_t(0)
    _check(lib().gomp_compress(src.ctypes.data if len(src) else None, len(src), out.ctypes.data, cap, ctypes.byref(n),
                               ctypes.byref(p)), "gomp_compress")
    return torch.from_numpy(out[: n.value].copy())


def compress_device(x, p=None, stream=None, **kw):
    """gomp_compress_device: compress a CUDA uint8 tensor on the GPU; returns the file as a CUDA uint8 tensor
    (identical to compress() of the same bytes and parameters)."""
    if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.uint8 and x.is_contiguous()):
        raise ValueError("compress_device() takes a contiguous CUDA uint8 tensor (no CPU fallback)")
    p = p or params(**kw)
    cap = lib().gomp_compress_bound(x.numel(), ctypes.byref(p))
    if cap == 0:
        raise GompError(-1, where="gomp_compress_bound")
    wsn = ctypes.c_size_t(0)
    _check(lib().gomp_compress_device_workspace_size(x.numel(), ctypes.byref(p), ctypes.byref(wsn)),
           "gomp_compress_device_workspace_size")
    out = torch.empty(cap, dtype=torch.uint8, device=x.device)
    ws = torch.empty(max(wsn.value, 16), dtype=torch.uint8, device=x.device)
    n = ctypes.c_size_t(0)
    _check(lib().gomp_compress_device(x.data_ptr() if x.numel() else None, x.numel(), out.data_ptr(), cap,
                                      ctypes.byref(n), ws.data_ptr(), ws.numel(), ctypes.byref(p),
                                      _stream_ptr(stream, x.device)), "gomp_compress_device")
    return out[: n.value]


def get_info(c):
    """gomp_get_info from the first 64 bytes of a file (host tensor / bytes; a CUDA tensor is read back)."""
    if isinstance(c, torch.Tensor):
        hdr = c[:64].cpu().numpy() if c.is_cuda else c[:64].numpy()
    else:
        hdr = _host_u8(c)[:64]
    hdr = np.ascontiguousarray(hdr, dtype=np.uint8)
    info = Info()
    _check(lib().gomp_get_info(hdr.ctypes.data, len(hdr), ctypes.byref(info)), "gomp_get_info")
    return info


def validate_tables(c):
    f = _host_u8(c)
    bad = ctypes.c_uint32(0)
    st = lib().gomp_validate_tables(f.ctypes.data, len(f), ctypes.byref(bad))
    if st:
        raise GompError(st, bad.value, where="gomp_validate_tables")


def workspace_size(info, n_blocks=0):
    n = ctypes.c_size_t(0)
    _check(lib().gomp_decompress_workspace_size(ctypes.byref(info), n_blocks, ctypes.byref(n)),
           "gomp_decompress_workspace_size")
    return n.value


def _stream_ptr(stream, device):
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return ctypes.c_void_p(s.cuda_stream)


def _strategy(strategy, stats, phase=None, huff=None):
    s = STRATEGIES[strategy] if isinstance(strategy, str) else int(strategy)
    s |= {None: 0, "decode": FLAG_DECODE_ONLY, "lz77": FLAG_LZ77_ONLY}[phase]
    s |= {None: 0, "thread": FLAG_HUFF_THREAD, "warp": FLAG_HUFF_WARP}[huff]
    return s | (FLAG_STATS if stats else 0)


def token_bytes(c):
    """Bytes of the Bit decoder's token stream for file c (host tensor/array): sum over blocks of 4 B per record
    + 1 B per literal (FORMAT.md block table; host arithmetic for reporting, no decoding)."""
    a = np.asarray(c if not isinstance(c, torch.Tensor) else c.cpu().numpy(), dtype=np.uint8)
    info = get_info(a)
    t = a[64:64 + 32 * info.n_blocks].view(np.uint32).reshape(-1, 8)
    return int(4 * t[:, 3].astype(np.int64).sum() + t[:, 4].astype(np.int64).sum())


def huff_variant(info):
    """Which Bit decoder the launcher picks (mirrors decompress_range): "warp" when the mean sub-block holds at
    least 8192 bits (kWarpMinAvgBits), else "thread"."""
    if not info.n_sub_total:
        return "thread"
    return "warp" if (info.file_len - info.payload_base) * 8 // info.n_sub_total >= 8192 else "thread"


def decompress_into(info, src, dst, workspace, strategy="auto", stream=None, first_block=0, n_blocks=None,
                    stats=False, phase=None, huff=None):
    """Enqueue gomp_decompress(_blocks) on `stream` (no synchronisation). src/dst/workspace: CUDA uint8
    tensors; dst receives block first_block at dst[0]. phase="decode"/"lz77" runs one kernel of a Bit
    decompression (profiling only, GOMP_FLAG_DECODE_ONLY / GOMP_FLAG_LZ77_ONLY); huff="thread"/"warp"
    forces the Bit decoder variant (testing, GOMP_FLAG_HUFF_THREAD / GOMP_FLAG_HUFF_WARP)."""
    for t in (src, dst, workspace):
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.uint8 and t.is_contiguous()):
            raise ValueError("decompress_into needs contiguous CUDA uint8 tensors (no CPU fallback)")
    sp = _stream_ptr(stream, src.device)
    nb = info.n_blocks - first_block if n_blocks is None else n_blocks
    _check(lib().gomp_decompress_blocks(ctypes.byref(info), first_block, nb, src.data_ptr(), src.numel(),
                                        dst.data_ptr(), dst.numel(), workspace.data_ptr(), workspace.numel(),
                                        _strategy(strategy, stats, phase, huff), sp), "gomp_decompress")


def read_error(workspace, stream=None):
    e = Error()
    _check(lib().gomp_decompress_error(workspace.data_ptr(), _stream_ptr(stream, workspace.device), ctypes.byref(e)),
           "gomp_decompress_error")
    return e


def read_stats(workspace, stream=None):
    s = Stats()
    _check(lib().gomp_decompress_stats(workspace.data_ptr(), _stream_ptr(stream, workspace.device), ctypes.byref(s)),
           "gomp_decompress_stats")
    return {"rounds": list(s.rounds), "bytes": list(s.bytes), "de_fallback_groups": s.de_fallback_groups}


def decompress(c, out=None, strategy="auto", stream=None, info=None, check=True, stats=False, return_stats=False,
               huff=None):
    """Decompress a Gompresso file held in a CUDA uint8 tensor; returns a CUDA uint8 tensor.
    check=True synchronises and raises GompError on a device-detected error."""
    if not (isinstance(c, torch.Tensor) and c.is_cuda):
        raise ValueError("decompress() takes a CUDA tensor (no CPU fallback); use .cuda()")
    info = info or get_info(c)
    if out is None:
        out = torch.empty(max(info.uncompressed_len, 1), dtype=torch.uint8, device=c.device)
    ws = torch.empty(workspace_size(info), dtype=torch.uint8, device=c.device)
    decompress_into(info, c, out, ws, strategy, stream, stats=stats or return_stats, huff=huff)
    if check:
        e = read_error(ws, stream)
        if e.status:
            raise GompError(e.status, e.block, e.detail, where="gomp_decompress")
    y = out[: info.uncompressed_len]
    if return_stats:
        return y, read_stats(ws, stream)
    return y


def decompress_host(c_host, out_host=None, strategy="auto", device=None, stream=None, bufs=None, info=None,
                    in_mode=False):
    """End-to-end path (gomp_decompress_host): host (pinned) compressed file -> host output, with the copies
    enqueued on the stream. Returns the host output tensor (synchronised, error-checked). in_mode=True is the
    paper's "In" mode: only the compressed file crosses the host link, the output stays on the
    device and the device tensor is returned."""
    device = torch.device(device or "cuda")
    info = info or get_info(c_host)
    if out_host is None:
        out_host = torch.empty(max(info.uncompressed_len, 1), dtype=torch.uint8, pin_memory=True)
    if bufs is None:
        bufs = (torch.empty(info.file_len, dtype=torch.uint8, device=device),
                torch.empty(max(info.uncompressed_len, 1), dtype=torch.uint8, device=device),
                torch.empty(workspace_size(info), dtype=torch.uint8, device=device))
    d_src, d_dst, ws = bufs
    sp = _stream_ptr(stream, device)
    _check(lib().gomp_decompress_host(ctypes.byref(info), c_host.data_ptr(), c_host.numel(),
                                      None if in_mode else out_host.data_ptr(), 0 if in_mode else out_host.numel(),
                                      d_src.data_ptr(), d_dst.data_ptr(), ws.data_ptr(), ws.numel(),
                                      _strategy(strategy, False), sp), "gomp_decompress_host")
    e = read_error(ws, stream)
    if e.status:
        raise GompError(e.status, e.block, e.detail, where="gomp_decompress_host")
    return d_dst[: info.uncompressed_len] if in_mode else out_host[: info.uncompressed_len]


def plan_shards(c_host, n_dev):
    """gomp_plan_shards: contiguous block ranges per device balanced by compressed bytes."""
    f = _host_u8(c_host)
    first = (ctypes.c_uint32 * (n_dev + 1))()
    _check(lib().gomp_plan_shards(f.ctypes.data, len(f), n_dev, first), "gomp_plan_shards")
    return list(first)


def shard_file(c_host, first_block, n_blocks):
    """gomp_shard_file: a standalone file (CPU torch.uint8 tensor) of blocks [first_block, first_block + n_blocks)
    with rebased tables; it decodes to bytes [first_block * block_size, ...) of the whole output."""
    f = _host_u8(c_host)
    n = ctypes.c_size_t(0)
    _check(lib().gomp_shard_file(f.ctypes.data, len(f), first_block, n_blocks, None, 0, ctypes.byref(n)),
           "gomp_shard_file")
    out = np.empty(n.value, dtype=np.uint8)
    _check(lib().gomp_shard_file(f.ctypes.data, len(f), first_block, n_blocks, out.ctypes.data, n.value,
                                 ctypes.byref(n)), "gomp_shard_file")
    return torch.from_numpy(out)


def decompress_sharded(c_host, devices, strategy="auto"):
    """Decompress one file across several GPUs of this process (blocks are independent,
    P:30-31): gomp_plan_shards splits the blocks into contiguous ranges balanced by compressed bytes; device d
    receives only the shard file of its range (gomp_shard_file: rebased tables + its payloads, host->device from
    pinned memory on its own stream), so its memory is O(shard), and decodes it. No collective, no gather:
    returns [(first_block, CUDA uint8 tensor of that range's output)] in device order."""
    f = _host_u8(c_host)
    info = get_info(f)
    devices = [torch.device(d) for d in devices]
    first = plan_shards(f, len(devices))
    outs, pending = [], []
    for d, dev in enumerate(devices):
        b0, b1 = first[d], first[d + 1]
        h = shard_file(f, b0, b1 - b0).pin_memory()
        sinfo = get_info(h)
        with torch.cuda.device(dev):
            stream = torch.cuda.Stream(dev)
            with torch.cuda.stream(stream):   # allocations and copies ordered on this device's stream
                src = torch.empty(h.numel(), dtype=torch.uint8, device=dev)
                out = torch.empty(max(sinfo.uncompressed_len, 1), dtype=torch.uint8, device=dev)
                ws = torch.empty(workspace_size(sinfo), dtype=torch.uint8, device=dev)
                src.copy_(h, non_blocking=True)
                decompress_into(sinfo, src, out, ws, strategy, stream)
            pending.append((dev, stream, ws, b0, src, h))   # buffers stay referenced until the stream syncs
            outs.append((b0, out[: sinfo.uncompressed_len]))
    for dev, stream, ws, b0, _, _ in pending:
        e = read_error(ws, stream)
        if e.status:   # the shard's block index, reported as the whole file's block index
            raise GompError(e.status, b0 + e.block, e.detail, where=f"decompress_sharded({dev})")
    return outs
