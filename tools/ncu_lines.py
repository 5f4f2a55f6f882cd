#!/usr/bin/env python
"""Per-CUDA-source-line warp-stall samples from an ncu report (needs -lineinfo):
   python tools/ncu_lines.py <rep> [kernel-substring] [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; ksub = sys.argv[2] if len(sys.argv) > 2 else ""; top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fn, hdr, src = None, None, {}
res = {}
for r in rows:
    if not r: continue
    if r[0] == "Function Name": fn = r[1]; continue
    if r[0] == "File Path": continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or fn is None or ksub not in fn: continue
    try:
        si = hdr.index("Warp Stall Sampling (All Samples)")
    except ValueError:
        continue
    if r[2] != "-":  # sass rows under a line: skip (line rows carry aggregates)
        continue
    d = res.setdefault(fn, [])
    reasons = {hdr[i]: int(float(r[i])) for i in range(len(hdr)) if hdr[i].startswith("stall_") and "Not Issued" not in hdr[i] and r[i] not in ("", "-") and float(r[i]) > 0}
    d.append((int(float(r[si] or 0)), r[0], r[1].strip()[:90], sorted(reasons.items(), key=lambda kv: -kv[1])[:3]))
for f, d in res.items():
    tot = sum(x[0] for x in d)
    print(f"== {f[:90]}  total samples {tot}")
    for s, ln, code, rs in sorted(d, key=lambda x: -x[0])[:top]:
        print(f"{s:8d} {100*s/max(tot,1):5.1f}% L{ln:>4} {code:90s} {rs}")
