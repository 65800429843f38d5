"""clock64 timeline of the projection kernel's CTA (0, 0) (development tool; SALS_TC_TRACE build)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2510_24273_b200 import sals
sh = dict(synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
cfg = sals.make_config(**sh)
B, s = sh["batch"], sh["seq"]
g = torch.Generator(device="cuda"); g.manual_seed(1)
ly = synth.gen_layer_torch(num_q_heads=sh["num_q_heads"], num_kv_heads=sh["num_kv_heads"], head_dim=128, rank=sh["rank"], batch=B, seq=s, generator=g)
seq = torch.full((B,), s, dtype=torch.int32, device="cuda")
ws = sals.alloc_workspace(sals.sals_workspace_bytes(cfg, B, s), "cuda")
out = torch.empty(B, sh["num_q_heads"] * 128, dtype=torch.bfloat16, device="cuda")
torch.cuda.synchronize()
for _ in range(3):
    sals.sals_append_decode(cfg, ly["U"], ly["k_new"], ly["v_new"], ly["q"], ly["latent"], ly["v"], seq, s, out, ws)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 16)()
sals._lib.sals_debug_proj_trace(buf)
t = np.array(buf[:8], dtype=np.int64)
names = ["start", "U_issued", "after_wait", "x_staged+U_landed", "fma_done", "cta_reduced", "cluster_sync1", "done"]
for i, n in enumerate(names):
    print(f"{n:20s} {(t[i] - t[0]) / 1000:8.2f} kcycles")
