"""Host cost of one sals_append_decode call at c2 (the eager e2e path): wall time per call
with the kernels enqueued (GPU far behind: host-bound measure), with every stage masked off
(validation, plan, tensor maps, Python marshalling only), and the Python-side marshalling."""
import sys, os, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2510_24273_b200 import sals
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
sh = dict(synth.CONFIGS[name])
cfg = sals.make_config(**sh)
B, s = sh["batch"], sh["seq"]
g = torch.Generator(device="cuda"); g.manual_seed(1)
L = 4
lys = [synth.gen_layer_torch(num_q_heads=sh["num_q_heads"], num_kv_heads=sh["num_kv_heads"], head_dim=128,
                             rank=sh["rank"], batch=B, seq=s, generator=g) for _ in range(L)]
seq = torch.full((B,), s, dtype=torch.int32, device="cuda")
ws = sals.alloc_workspace(sals.sals_workspace_bytes(cfg, B, s), "cuda")
out = torch.empty(B, sh["num_q_heads"] * 128, dtype=torch.bfloat16, device="cuda")
def call(ly):
    sals.sals_append_decode(cfg, ly["U"], ly["k_new"], ly["v_new"], ly["q"], ly["latent"], ly["v"], seq, s, out, ws)
for ly in lys: call(ly)
torch.cuda.synchronize()
N = 400
def timed(tag):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(N): call(lys[i % L])
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{tag:28s} host {1e6 * (t1 - t0) / N:7.2f} us/call   wall incl. drain {1e6 * (t2 - t0) / N:7.2f} us/call")
timed("full")
old = sals._lib.sals_profile_stage_mask(0)
timed("no kernels (mask 0)")
sals._lib.sals_profile_stage_mask(old)
t0 = time.perf_counter()
for i in range(N):
    ly = lys[i % L]
    args = (ctypes.byref(cfg), sals._p(ly["U"]), sals._p(ly["k_new"]), sals._p(ly["v_new"]), sals._p(ly["q"]),
            sals._p(ly["latent"]), sals._p(ly["v"]), sals._stream(None))
t1 = time.perf_counter()
print(f"{'python marshalling only':28s} host {1e6 * (t1 - t0) / N:7.2f} us/call")
t0 = time.perf_counter()
for i in range(N): sals._stream(None)
t1 = time.perf_counter()
print(f"{'torch current_stream':28s} host {1e6 * (t1 - t0) / N:7.2f} us/call")
