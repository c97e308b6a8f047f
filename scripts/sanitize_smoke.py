"""Small runs of every device kernel, for compute-sanitizer (one tool per gpurun call)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_02692_b200 as X  # noqa: E402
import synth  # noqa: E402
from oracle import matrices as mx  # noqa: E402
from oracle import rs  # noqa: E402

n, p, B, S = 10, 4, 4224, 3            # 4224 = 33 x 128: ragged tiles
og = mx.coding_matrix(n, p)
G = X.xslp_coding_matrix(n, p)
bits = X.xslp_encode_bitmatrix(G, n, p)
data = np.stack([synth.stripe_data(9, s, n, B) for s in range(S)])
din = torch.from_numpy(data).cuda()
ok = True
for kern, extra in [("straight", {}), ("tma", {}), ("pipe", dict(threads=64)), ("interp", {}),
                    ("straight", dict(layout="byte"))]:
    prog = X.xslp_compile(bits, kernel=kern, **extra)
    dout = torch.zeros((S, p, B), dtype=torch.uint8, device="cuda")
    X.xslp_encode_batch(prog, X.block_table(din, S, n, B), X.block_table(dout, S, p, B), S, B)
    torch.cuda.synchronize()
    for s in range(S):
        want = (rs.bytewise_apply(og[n:], data[s]) if extra.get("layout") == "byte"
                else rs.encode(og, n, data[s]))
        ok &= bool((dout[s].cpu().numpy() == want).all())
    print(kern, extra, ok, flush=True)
# interpreter with LDG staging (strip not a multiple of 16 bytes) and one-stripe entries
B2 = 4128                                  # strip 516 B: 16-byte TMA not possible
d2 = torch.from_numpy(synth.stripe_data(3, 0, n, B2)).cuda()
for kern in ("interp", "straight"):
    prog = X.xslp_compile(bits, kernel=kern)
    o2 = torch.zeros((p, B2), dtype=torch.uint8, device="cuda")
    X.xslp_encode(prog, [d2[j] for j in range(n)], [o2[i] for i in range(p)], B2)
    torch.cuda.synchronize()
    ok &= bool((o2.cpu().numpy() == rs.encode(og, n, synth.stripe_data(3, 0, n, B2))).all())
    print("one", kern, ok, flush=True)
# codec
c = X.Codec(10, 4)
ln = 100001
buf = torch.from_numpy(np.frombuffer(os.urandom(ln), dtype=np.uint8).copy()).cuda()
sh = torch.zeros((14, c.block_bytes(ln)), dtype=torch.uint8, device="cuda")
c.encode(buf, ln, sh)
out = torch.zeros(ln, dtype=torch.uint8, device="cuda")
c.decode(sh, [0, 3, 11, 12], ln, out)
torch.cuda.synchronize()
ok &= bool(torch.equal(out, buf))
print("codec", ok)
sys.exit(0 if ok else 1)
