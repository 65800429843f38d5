"""Stage-by-stage GPU vs oracle diagnostics (development tool)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from oracle import sals_oracle as O
from tests import harness as H
from paper_2510_24273_b200 import sals

def run(shape, B, seqs, **kw):
    cfg, host, gpu = H.run_sals(shape, B, seqs, **kw)
    oc = H.oracle_cfg(shape, kw.get("sink", 0), kw.get("recent", 0))
    orc = O.decode(oc, host["U"], host["q"], host["latent"], host["v"], host["seq_len"])
    for b in range(B):
        s = int(host["seq_len"][b])
        e = np.abs(gpu["scores"][b, :s] - orc["scores"][b])
        print(f"b={b} s={s} score maxerr={e.max():.3e} at {e.argmax()} gpu={gpu['scores'][b,:6]} orc={orc['scores'][b][:6]}")
        gs = gpu["sel"][b]; gs = gs[gs >= 0]
        print("  sel gpu[:12]", gs[:12], "orc[:12]", orc["sel"][b][:12], "n", len(gs), len(orc["sel"][b]),
              "symdiff", len(set(gs.tolist()) ^ set(orc["sel"][b].tolist())))
    forced = [gpu["sel"][b][gpu["sel"][b] >= 0].astype(np.int64) for b in range(B)]
    of = O.decode(oc, host["U"], host["q"], host["latent"], host["v"], host["seq_len"], forced_selection=forced)
    e = np.abs(gpu["out"] - of["y"])
    print(f"  out maxerr (forced) {e.max():.3e} mean-rel {e.sum()/np.abs(of['y']).sum():.3e}")
    return cfg, host, gpu, orc

if __name__ == "__main__":
    C = synth.CONFIGS
    path = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    if path == 2:
        sh = dict(C["c3"]); sh.update(num_q_heads=16, num_kv_heads=4, rank=256, score_rank=128, top_k=200)
        run(sh, 3, [700, 2049, 300], path=2)
        sh = dict(C["c2"]); sh.update(rank=512, score_rank=256, top_k=512)
        run(sh, 2, [4096, 1000], path=2)
        sys.exit(0)
    run(dict(C["c1"]), 1, [256])
    sh = dict(C["c2"]); sh.update(num_q_heads=4, num_kv_heads=4, rank=64, score_rank=32, top_k=40)
    run(sh, 2, [5000, 3000], path=path)
    sh = dict(C["c3"]); sh.update(num_q_heads=16, num_kv_heads=4, rank=256, score_rank=128, top_k=200)
    run(sh, 3, [700, 2049, 300], path=path)
