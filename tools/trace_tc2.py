import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2510_24273_b200 import sals
sh = dict(synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
VB, Z = int(os.environ.get("V_BITS", "0")), int(os.environ.get("RECENT", "0"))
cfg = sals.make_config(**sh, v_bits=VB, recent=Z)
B, s = sh["batch"], sh["seq"]
g = torch.Generator(device="cuda"); g.manual_seed(1)
ly = synth.gen_layer_torch(num_q_heads=sh["num_q_heads"], num_kv_heads=sh["num_kv_heads"], head_dim=128, rank=sh["rank"], batch=B, seq=s, generator=g)
seq = torch.full((B,), s, dtype=torch.int32, device="cuda")
ws = sals.alloc_workspace(sals.sals_workspace_bytes(cfg, B, s), "cuda")
out = torch.empty(B, sh["num_q_heads"] * 128, dtype=torch.bfloat16, device="cuda")
vbuf = ly["v"]
if VB:   # synthetic quantised rows (valid bf16 parameters), as in bench.py
    nkv, nbc, rb = sh["num_kv_heads"], 128 * VB // 8, sals.sals_v_row_bytes(cfg)
    vbuf = torch.randint(0, 256, (sals.sals_v_cache_bytes(cfg, B, s),), dtype=torch.uint8, device="cuda")
    vbuf[:B * s * rb].view(B, s, nkv, nbc + 16)[..., nbc:] = torch.tensor([0.05, -0.4], dtype=torch.bfloat16, device="cuda").view(torch.uint8).repeat(4)
    if Z:
        vbuf[B * s * rb:].view(B, Z, nkv, 144)[..., 128:] = torch.tensor([0.003, -0.4], dtype=torch.bfloat16, device="cuda").view(torch.uint8).repeat(4)
for _ in range(3):
    sals.sals_decode(cfg, ly["U"], ly["q"], ly["latent"], vbuf, seq, s, out, ws)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 128)()
sals._lib.sals_debug_tc_trace(buf)
t = np.array(buf[:], dtype=np.int64)
t0 = t[80]
names = {0: "mma_start", 88: "pfull0(cg2)", 8: "mma_commit", 16: "epi_tfull", 24: "epi_logits", 32: "epi_vfull", 40: "epi_pvdone", 64: "a_first_iss", 72: "a_last_iss"}
for base, nm in names.items():
    print(f"{nm:12s}", " ".join(f"{(t[base+i]-t0)/1000:8.2f}" for i in range(4)), " kcycles")
print("relay(cg2,t0) ", " ".join(f"{(t[96+i]-t0)/1000:7.2f}" for i in range(8)))
print("after_wait", (t[82]-t0)/1000, "end", (t[81]-t0)/1000)
