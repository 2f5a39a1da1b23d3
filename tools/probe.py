"""Quick timing probe of the GPU engine (dev tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2104_09164_b200.ckks.engine import CkksBackend
from paper_2104_09164_b200.ckks.params import gen_params
from paper_2104_09164_b200.fastpath import compile_pipeline, encrypt_input, run_pipeline, dec_logits
from paper_2104_09164_b200.model import net_by_name, collapse_layers, make_random_model, make_random_input, infer_clear
from paper_2104_09164_b200.modelenc import ModelEncoder

def run(net, mode, strat, B, reps=2):
    prof = "fast-hear" if mode == "fast" else "hear"
    shape = net_by_name(net)
    cpar = collapse_layers(make_random_model(shape, 1), shape)
    t = time.time(); be = CkksBackend(gen_params(prof), seed=0); torch.cuda.synchronize(); tk = time.time()-t
    cp = compile_pipeline(shape, mode, strat, be.params)
    t = time.time(); be.ensure_rotation_keys(cp.rotations); torch.cuda.synchronize(); tr = time.time()-t
    enc = ModelEncoder(cp, cpar, be)
    t = time.time(); enc.prepare(); torch.cuda.synchronize(); te = time.time()-t
    x = np.stack([make_random_input(shape, 2 + i) for i in range(B)])
    ct = encrypt_input(x, cp, be)
    times = []
    for r in range(reps):
        torch.cuda.synchronize(); t = time.time()
        out = run_pipeline(enc, ct, be)
        torch.cuda.synchronize(); times.append(time.time() - t)
    lg = dec_logits(out, cp, be)
    ref = np.stack([infer_clear(cpar, xi) for xi in x])
    print(f"{net} {mode} {strat} B={B}: keygen {tk:.2f}s rotkeys {tr:.2f}s encode {te:.2f}s "
          f"eval {[round(v,3) for v in times]} s -> {B/min(times):.1f} inf/s  maxerr {np.abs(lg-ref).max():.2e} "
          f"mem {torch.cuda.max_memory_allocated()/2**30:.1f} GiB", flush=True)
    del be, enc, ct, out
    torch.cuda.empty_cache(); torch.cuda.reset_peak_memory_stats()

for spec in sys.argv[1:]:
    net, mode, strat, B = spec.split(":")
    run(net, mode, strat, int(B))
