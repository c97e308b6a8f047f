"""Quick bounded check of the persistent TMA pipeline kernel before the full suite."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2108_02692_b200 as X
import synth
from oracle import matrices as mx, rs
n, p, B, S = 10, 4, 9600, 5
g = X.xslp_coding_matrix(n, p)
prog = X.xslp_compile(X.xslp_encode_bitmatrix(g, n, p), kernel="pipe")
data = np.stack([synth.stripe_data(4, s, n, B) for s in range(S)])
din = torch.from_numpy(data).cuda()
dout = torch.zeros((S, p, B), dtype=torch.uint8, device="cuda")
X.xslp_encode_batch(prog, X.block_table(din, S, n, B), X.block_table(dout, S, p, B), S, B)
torch.cuda.synchronize()
og = mx.coding_matrix(n, p)
ok = all((dout[s].cpu().numpy() == rs.encode(og, n, data[s])).all() for s in range(S))
print("pipe smoke", "OK" if ok else "MISMATCH", prog.stats()["regs_pipe"])
sys.exit(0 if ok else 1)
