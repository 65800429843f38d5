"""Per-CTA globaltimer stamps of the fused kernel (build with -DSALS_TC_CTATIME):
start / after the PDL wait / last MMA commit / end of every CTA of the last launch
of a 32-layer append_decode graph-free loop, relative to the earliest start."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2510_24273_b200 import sals
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
sh = dict(synth.CONFIGS[name])
cfg = sals.make_config(**sh)
B, s = sh["batch"], sh["seq"]
g = torch.Generator(device="cuda"); g.manual_seed(1)
L = 8
lys = [synth.gen_layer_torch(num_q_heads=sh["num_q_heads"], num_kv_heads=sh["num_kv_heads"], head_dim=128,
                             rank=sh["rank"], batch=B, seq=s, generator=g) for _ in range(L)]
seq = torch.full((B,), s, dtype=torch.int32, device="cuda")
ws = sals.alloc_workspace(sals.sals_workspace_bytes(cfg, B, s), "cuda")
out = torch.empty(B, sh["num_q_heads"] * 128, dtype=torch.bfloat16, device="cuda")
for ly in lys:   # full calls first: the workspace then holds a valid selection
    sals.sals_decode(cfg, ly["U"], ly["q"], ly["latent"], ly["v"], seq, s, out, ws)
torch.cuda.synchronize()
mask = int(os.environ.get("MASK", "-1"))   # e.g. 8: only the fused kernel (back-to-back launches)
if mask >= 0:
    sals._lib.sals_profile_stage_mask(mask)
for rep in range(3):
    for ly in lys:
        sals.sals_decode(cfg, ly["U"], ly["q"], ly["latent"], ly["v"], seq, s, out, ws)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (1024 * 4))()
assert sals._lib.sals_debug_tc_ctatime(buf) == 0
t = np.array(buf[:], dtype=np.int64).reshape(1024, 4)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
r = (t - t0) / 1000.0
print(f"{name}: {len(r)} CTAs (us from the first start)")
for k, nm in enumerate(["start", "after_wait", "last_mma", "end"]):
    v = r[:, k]
    print(f"  {nm:11s} min {v.min():7.2f} p10 {np.percentile(v,10):7.2f} p50 {np.median(v):7.2f} p90 {np.percentile(v,90):7.2f} max {v.max():7.2f}")
d = r[:, 3] - r[:, 1]
print(f"  busy(end-after_wait) min {d.min():.2f} p50 {np.median(d):.2f} max {d.max():.2f}")
order = np.argsort(r[:, 3])[-5:]
print("  slowest CTAs (start, wait, mma, end):", [tuple(np.round(r[i], 2)) for i in order])
