"""Diagnostic: engine vs oracle per tier split (tiny fp32)."""
import sys, traceback
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import oracle_bindings as ob
import paper_2512_17570_b200 as gs
ADAM = dict(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.0)
g, M, iters = ob.TINY, 4, int(sys.argv[1]) if len(sys.argv) > 1 else 2
for split, alpha, tier in [((1,1,1),0,0), ((0,1,1),0,0), ((1,0,1),0,0), ((1,1,0),0,0), ((1,1,0),0,2), ((0,0,0),0,0)]:
    try:
        model = gs.ModelSpec(g.n_layers, g.hidden, g.heads, g.seq, g.mb_size, 4, 4, 3, 1)
        plan = gs.build_vertical(model, M, gs.StorageSplit(*split), alpha)
        eng = gs.Engine(plan, model, g.vocab, gs.AdamConfig(**ADAM), seed=42, nvme_dir="/tmp", opt_tier=tier)
        tok = ob.make_tokens(g, iters, M)
        rep = eng.run(tok); eng.flush(); L, F = eng.read_params(); eng.close()
        l0, f0 = ob.init_params(g)
        rl, RL, RF, _, _ = ob.train(g, ADAM, M, plan.as_dict(), tok, l0, f0)
        bad = np.abs(L - RL) > 1e-5 * (1 + np.abs(RL))
        per_layer = bad.mean(1)
        idx = [np.nonzero(bad[l])[0] for l in range(g.n_layers)]
        print(split, alpha, tier, "loss", np.array(rep.losses) - rl, "bad frac/layer", per_layer,
              "first/last bad", [(int(i[0]), int(i[-1])) if len(i) else None for i in idx],
              "fixed rel", np.linalg.norm(F - RF) / np.linalg.norm(RF), "ext", rep.extension.sum(1), flush=True)
    except Exception:
        traceback.print_exc()
