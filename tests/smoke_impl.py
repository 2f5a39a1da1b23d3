"""__graft_entry__.smoke(): one tiny encrypted evaluation on cuda:0 checked
against the CPU oracle (toy parameters, toy network)."""

import numpy as np


def run_smoke():
    import torch
    from oracle.cpu_engine import OracleCkks
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params
    from paper_2104_09164_b200.fastpath import compile_pipeline, infer
    from paper_2104_09164_b200.model import (NetworkShape, collapse_layers, infer_clear,
                                             make_random_input, make_random_model)
    from paper_2104_09164_b200.modelenc import ModelEncoder
    assert torch.cuda.is_available(), "smoke needs cuda:0"
    shape = NetworkShape(1, 32, 15, (4, 8, 16), 4)
    cpar = collapse_layers(make_random_model(shape, 3), shape)
    x = make_random_input(shape, 4)
    ps = gen_params("toy-fast")
    gpu = CkksBackend(ps, seed=5, device="cuda:0")
    cpu = OracleCkks(ps, seed=5)
    cp = compile_pipeline(shape, "fast", "giant", ps)
    gpu.ensure_rotation_keys(cp.rotations)
    cpu.ensure_rotation_keys(cp.rotations)
    # key material bit-exact against the oracle
    assert np.array_equal(gpu.keys.relin.b.cpu().numpy().view(np.uint64), cpu.keys.relin.b)
    lg_g, cnt_g, _ = infer(cpar, x, "fast", "giant", gpu, encoder=ModelEncoder(cp, cpar, gpu))
    lg_c, cnt_c, _ = infer(cpar, x, "fast", "giant", cpu, encoder=ModelEncoder(cp, cpar, cpu))
    torch.cuda.synchronize()
    scale = max(np.abs(lg_c).max(), 1e-12)
    err = np.abs(lg_g - lg_c).max()
    assert err <= 1e-3 * scale, (lg_g, lg_c)
    assert int(np.argmax(lg_g)) == int(np.argmax(lg_c))
    assert cnt_g.as_dict() == cnt_c.as_dict()
    clear = infer_clear(cpar, x)
    print(f"smoke ok: gpu vs oracle max|d| = {err:.3e}, vs clear {np.abs(lg_g - clear).max():.3e}")


if __name__ == "__main__":
    run_smoke()
