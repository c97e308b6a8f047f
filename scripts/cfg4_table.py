"""Markdown table of the cfg4 sweep (scripts/cfg4_sweep.sh output)."""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.strip()]
print("| p | block | program | GB/s data | roofline frac | #xor | #M | regs (LDG/pipe) | kernel |")
print("|---|---|---|---|---|---|---|---|---|")
for d in rows:
    if "failed" in d:
        print(f"| failed: {d['failed']} |||||||||")
        continue
    c = d["config"]
    s = c["slp"]
    print(f"| {c['p']} | {c['block_bytes'] // 1024} KiB | {c['program']} | {d['value']:.0f} | "
          f"{d['roofline']['frac']:.3f} | {s['xor_count']} | {s['mem_count']} | "
          f"{s['regs']}/{s['regs_pipe']} | {d['roofline']['kernel']} |")
