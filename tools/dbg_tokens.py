"""Dev helper: compare the Bit decoder's token buffer with the oracle's sequences, block by block."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch, datagen, oracle, paper_1606_00519_b200 as gomp
kind = sys.argv[1] if len(sys.argv) > 1 else "wiki"
bs = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
k = int(sys.argv[3]) if len(sys.argv) > 3 else 16
x = datagen.wiki(1_100_003, seed=1) if kind == "wiki" else datagen.text(1 << 20, seed=1)
c = gomp.compress(x, mode="bit", de=True, block_size=bs, sub_block_seqs=0, sub_blocks_per_block=k)
info = gomp.get_info(c)
d = c.cuda(); out = torch.empty(info.uncompressed_len, dtype=torch.uint8, device="cuda")
ws = torch.zeros(gomp.workspace_size(info), dtype=torch.uint8, device="cuda")
gomp.decompress_into(info, d, out, ws, phase="decode")
e = gomp.read_error(ws); print("err", e.status, e.block, hex(e.detail))
wsn = ws.cpu().numpy(); cn = c.numpy()
stride = (info.max_block_tokens + 15) // 16 * 16
import struct
for b in range(info.n_blocks):
    seqs = oracle.block_sequences(cn, b)
    off, plen, n_seq, n_lit, sf, S, ns = struct.unpack_from("<QIIIIII", cn.tobytes(), 64 + 32 * b)
    tok = wsn[1024 + b * stride: 1024 + b * stride + 4 * n_seq + n_lit]
    recs = tok[:4 * n_seq].view(np.uint32)
    mm = info.min_match
    exp = np.array([(l | ((L - mm + 1) << 10 if L else 0) | ((d - 1) << 16 if L else 0)) for l, L, d in seqs], dtype=np.uint32)
    bad = np.flatnonzero(recs != exp)
    if len(bad):
        i = bad[0]
        print(f"block {b}: {len(bad)} bad records of {n_seq}; first {i} (sub-block {i // S}, idx in sub {i % S}) got {recs[i]:#x} exp {exp[i]:#x} (lit {recs[i]&1023} vs {exp[i]&1023})")
        print("   next bad:", bad[:10])
        break
else:
    print("all records match")
if len(bad):
    got = recs[i:i + 6]
    for sh in range(-40, 41):
        j = i + sh
        if 0 <= j and j + 6 <= len(exp) and np.array_equal(exp[j:j + 6] & ~np.uint32(1023), got & ~np.uint32(1023)):
            print("got[i:i+6] == exp shifted by", sh)
    print("got", [hex(v) for v in recs[i - 2:i + 4]])
    print("exp", [hex(v) for v in exp[i - 2:i + 4]])
dbg = out[:2048].cpu().numpy().view(np.uint32).reshape(32, 16)
print("lane on merged nlen0 nlen lits0 lits t_start e_pos exit_lane exit_idx recoff n_it lead runin cap c")
for l in range(32):
    print(l, [int(v) for v in dbg[l]])
