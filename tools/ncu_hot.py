"""Top source lines by warp-stall samples and stall reasons from an ncu report."""
import csv, subprocess, sys
rep = sys.argv[1]
KF = (["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []) + (["-s", sys.argv[4], "-c", "1"] if len(sys.argv) > 4 else [])
raw = subprocess.run(["ncu", "-i", rep, *KF, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, vals = rows[0], rows[2]
items = []
for i, h in enumerate(hdr):
    if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
        try: items.append((float(vals[i]), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError: pass
print("stalls:", ", ".join(f"{h}={int(v)}" for v, h in sorted(items, reverse=True)[:8]))
for w in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
          "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
          "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]:
    for i, h in enumerate(hdr):
        if h == w or (h.startswith(w) and "pct" in w):
            print(f"  {h} = {vals[i]} {rows[1][i]}")
src = subprocess.run(["ncu", "-i", rep, *KF, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, fb = {}, None
for r in csv.reader(src.splitlines()):
    if r and r[0] == "File Path": fb = r[1].split("/")[-1]; continue
    if len(r) < 5 or r[0] in ("", "Line No"): continue
    try: agg[(fb, r[0], r[1][:90])] = int(r[4] or 0)
    except ValueError: pass
tot = sum(agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{v:6d} {100*v/tot:5.1f}%  {k[0]}:{k[1]}  {k[2]}")
