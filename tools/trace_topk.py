import sys, os, ctypes
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
for _ in range(3):
    sals.sals_decode(cfg, ly["U"], ly["q"], ly["latent"], ly["v"], seq, s, out, ws)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 32)()
sals._lib.sals_debug_topk_hist_trace(buf)
t = np.array(buf[:], dtype=np.int64)
names = ["start", "digit0", "staged", "bar1", "landed", "select", "counts", "end"]
for i, n in enumerate(names):
    print(f"{n:8s} {(t[i]-t[0])/1000:8.2f} kcyc")
