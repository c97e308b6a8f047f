"""Dispatch probe (round 2): a direct-threaded register-machine interpreter in PTX.

Every thread owns W words per SLP variable; NS register slots R_i (static register names inside
the handlers) and an accumulator; ops come warp-uniformly from shared memory (one u32 each:
handler index | shared row offset << 9), prefetched D ahead; each handler ends with its own
`brx.idx` through one branch table.  Writes probe_<NS>_<W>_<D>.ptx; scripts/dispatch_host.cu
loads the cubin and reports warp-ops per clock per SM on random programs.
"""
import sys

NS = int(sys.argv[1]) if len(sys.argv) > 1 else 32
W = int(sys.argv[2]) if len(sys.argv) > 2 else 2
D = int(sys.argv[3]) if len(sys.argv) > 3 else 2
OUT = sys.argv[4] if len(sys.argv) > 4 else f"/tmp/probe_{NS}_{W}_{D}.ptx"

H = []  # (name, body lines)
for i in range(NS):
    H.append((f"XR{i}", [f"xor.b32 %a{w}, %a{w}, %r{i}_{w};" for w in range(W)]))
for i in range(NS):
    H.append((f"ST{i}", [f"mov.b32 %r{i}_{w}, %a{w};" for w in range(W)]))
for i in range(NS):
    H.append((f"LD{i}", [f"mov.b32 %a{w}, %r{i}_{w};" for w in range(W)]))
vec = {1: "", 2: ".v2", 4: ".v4"}[W]
tmp = ", ".join(f"%t{w}" for w in range(W))
tmpb = "{" + tmp + "}" if W > 1 else tmp
accb = "{" + ", ".join(f"%a{w}" for w in range(W)) + "}" if W > 1 else "%a0"
ld = [f"add.u32 %ad, %arg, %tb;", f"ld.shared{vec}.u32 {tmpb}, [%ad];"]
H.append(("XS", ld + [f"xor.b32 %a{w}, %a{w}, %t{w};" for w in range(W)]))
H.append(("LS", [f"add.u32 %ad, %arg, %tb;", f"ld.shared{vec}.u32 {accb}, [%ad];"]))
H.append(("SS", [f"add.u32 %ad, %arg, %tb;", f"st.shared{vec}.u32 [%ad], {accb};"]))
for i in range(NS):
    H.append((f"XRS{i}", ld + [f"xor.b32 %a{w}, %a{w}, %t{w};" for w in range(W)]
              + [f"xor.b32 %a{w}, %a{w}, %r{i}_{w};" for w in range(W)]))
H.append(("END", None))
NH = len(H)

L = []
e = L.append
e(".version 8.7\n.target sm_100a\n.address_size 64\n")
e(".extern .shared .align 16 .b8 smem[];\n")
e(".visible .entry probe(.param .u64 p_code, .param .u32 p_ncode, .param .u32 p_iters, "
  ".param .u64 p_out, .param .u64 p_cyc)\n{")
e(f".reg .b32 %r<{NS}>;")  # unused base decl
for i in range(NS):
    e(".reg .b32 " + ", ".join(f"%r{i}_{w}" for w in range(W)) + ";")
e(".reg .b32 " + ", ".join(f"%a{w}" for w in range(W)) + ";")
e(".reg .b32 " + ", ".join(f"%t{w}" for w in range(W)) + ";")
e(".reg .b32 %op, %h, %arg, %ad, %tb, %pc, %pc0, %it, %niter, %ttid, %tntid, %i, %x, %sbase, %nc, %rows;")
e(".reg .b32 " + ", ".join(f"%q{k}" for k in range(1, D + 1)) + ";")
e(".reg .b64 %gp, %ga, %c0, %c1, %cd, %o64;")
e(".reg .pred %p;")
e("ld.param.u64 %gp, [p_code]; ld.param.u32 %nc, [p_ncode]; ld.param.u32 %niter, [p_iters];")
e("mov.u32 %ttid, %tid.x; mov.u32 %tntid, %ntid.x; mov.u32 %sbase, smem;")
# copy code
e("mov.u32 %i, %ttid;\nCP: setp.ge.u32 %p, %i, %nc; @%p bra CPD;")
e("mul.wide.u32 %ga, %i, 4; add.u64 %ga, %ga, %gp; ld.global.u32 %x, [%ga];")
e("shl.b32 %ad, %i, 2; add.u32 %ad, %ad, %sbase; st.shared.u32 [%ad], %x;")
e("add.u32 %i, %i, %tntid; bra CP;\nCPD:")
e("shl.b32 %rows, %nc, 2; add.u32 %rows, %rows, %sbase; add.u32 %rows, %rows, 15; and.b32 %rows, %rows, -16;")
e(f"mul.lo.u32 %tb, %ttid, {4 * W}; add.u32 %tb, %tb, %rows;")
# fill 64 rows
e(f"mov.u32 %i, %ttid; mul.lo.u32 %x, %tntid, {64 * W};")
e("FL: setp.ge.u32 %p, %i, %x; @%p bra FLD;")
e("shl.b32 %ad, %i, 2; add.u32 %ad, %ad, %rows; mul.lo.u32 %h, %i, -1640531535; st.shared.u32 [%ad], %h;")
e("add.u32 %i, %i, %tntid; bra FL;\nFLD: bar.sync 0;")
for i in range(NS):
    for w in range(W):
        e(f"add.u32 %r{i}_{w}, %ttid, {i * 7 + w};")
for w in range(W):
    e(f"mov.u32 %a{w}, 0;")
e("mov.u32 %it, 0;")
e("mov.u64 %c0, %clock64;")
e("START: mov.u32 %pc, %sbase;")
for k in range(1, D + 1):
    e(f"ld.shared.u32 %q{k}, [%pc]; add.u32 %pc, %pc, 4;")

tbl = "tbl: .branchtargets " + ", ".join(f"H_{n}" for n, _ in H) + ";"
e(tbl)


def dispatch():
    out = ["mov.b32 %op, %q1;"]
    for k in range(1, D):
        out.append(f"mov.b32 %q{k}, %q{k + 1};")
    out.append(f"ld.shared.u32 %q{D}, [%pc]; add.u32 %pc, %pc, 4;")
    out.append("and.b32 %h, %op, 511; shr.u32 %arg, %op, 9;")
    out.append("brx.idx %h, tbl;")
    return out


for ln in dispatch():
    e(ln)
for name, body in H:
    e(f"H_{name}:")
    if body is None:
        e("add.u32 %it, %it, 1; setp.lt.u32 %p, %it, %niter; @%p bra START;")
        e("bra DONE;")
        continue
    for ln in body:
        e(ln)
    for ln in dispatch():
        e(ln)
e("DONE: mov.u64 %c1, %clock64; sub.s64 %cd, %c1, %c0;")
e("mov.u32 %x, 0;")
for i in range(NS):
    for w in range(W):
        e(f"xor.b32 %x, %x, %r{i}_{w};")
for w in range(W):
    e(f"xor.b32 %x, %x, %a{w};")
e("ld.param.u64 %o64, [p_out]; mov.u32 %i, %ctaid.x; mad.lo.u32 %i, %i, %tntid, %ttid;")
e("mul.wide.u32 %ga, %i, 4; add.u64 %ga, %ga, %o64; st.global.u32 [%ga], %x;")
e("setp.ne.u32 %p, %ttid, 0; @%p bra EXIT;")
e("ld.param.u64 %o64, [p_cyc]; mov.u32 %i, %ctaid.x; mul.wide.u32 %ga, %i, 8; add.u64 %ga, %ga, %o64;")
e("st.global.u64 [%ga], %cd;")
e("EXIT: ret;\n}")
open(OUT, "w").write("\n".join(L) + "\n")
# handler indices for the host
print(f"NH={NH} XR=0 ST={NS} LD={2 * NS} XS={3 * NS} LS={3 * NS + 1} SS={3 * NS + 2} "
      f"XRS={3 * NS + 3} END={4 * NS + 3}")
