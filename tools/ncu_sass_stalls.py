"""Per-SASS-instruction warp-stall samples of one kernel in an ncu report, grouped
into regions delimited by barrier / mbarrier-wait instructions (development tool).
  python tools/ncu_sass_stalls.py report.ncu-rep [min_samples]"""
import csv, subprocess, sys
rep = sys.argv[1]
mins = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ia, isrc, isamp = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
reasons = [(i, h[6:]) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
base = None
region, reg_tot, reg_r = 0, 0, {}
tot = 0
lines = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    a = int(r[ia], 16)
    base = a if base is None else base
    src = r[isrc].strip()
    s = int(r[isamp] or 0)
    tot += s
    rs = sorted(((int(r[i] or 0), n) for i, n in reasons), reverse=True)[:3]
    lines.append((a - base, src, s, rs))
print("total samples", tot)
acc, acc_r, start = 0, {}, 0
def flush(end, label):
    global acc, acc_r
    if acc:
        top = sorted(acc_r.items(), key=lambda kv: -kv[1])[:5]
        print(f"--- region {start:#07x}-{end:#07x} ({label}): {acc} samples {100*acc/tot:.1f}%  " + ", ".join(f"{n}={v}" for n, v in top))
    acc, acc_r = 0, {}
for off, src, s, rs in lines:
    acc += s
    for v, n in rs:
        acc_r[n] = acc_r.get(n, 0) + v
    if s >= mins:
        print(f"  {off:#07x} {s:6d}  {src[:60]:60s} " + " ".join(f"{n}={v}" for v, n in rs if v))
    if "BAR.SYNC" in src or "PHASECHK" in src or "EXIT" in src:
        flush(off, src.split()[0] if src else "")
        start = off
flush(lines[-1][0], "end")
