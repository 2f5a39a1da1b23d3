"""Streaming latency (BASELINE config 4): a synthetic 30 fps skeleton stream
(15 joints x 2 coords, smoothed random walk in [-1, 1], 18000 frames) cut
into 32-frame windows with stride 8; every window is normalized (ingest),
encrypted, evaluated by the encrypted network (CUDA-graph replay, batch 1)
and decrypted.  The network is BASELINE's config-0 temporal network
(tcn.py: conv1d k=8 / 32 filters / stride 2, square, average pool, FC to 5)
by default; `--net 1d-w64` runs a reference HEAR network instead.  Reports
p50/p99 per-window latency on one GPU, split into the client side (ingest +
encrypt + decrypt) and the server side (encrypted evaluation), plus the
batched throughput over the same windows.

    python tools/stream_bench.py [--frames 18000] [--net config0|1d-w64] [--strategy full]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2104_09164_b200 import ingest
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params
    from paper_2104_09164_b200.fastpath import (GraphedPipeline, compile_pipeline, dec_logits,
                                                encrypt_input)
    from paper_2104_09164_b200.model import (collapse_layers, infer_clear, make_random_model,
                                             net_by_name)
    from paper_2104_09164_b200.modelenc import ModelEncoder

    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=18000)
    ap.add_argument("--net", default="config0")
    ap.add_argument("--strategy", default="full")
    ap.add_argument("--batch", type=int, default=64)
    args = ap.parse_args()
    be = CkksBackend(gen_params("fast-hear"), seed=0)
    if args.net.startswith("config"):
        from paper_2104_09164_b200 import tcn
        shape = tcn.tcn_by_name(args.net)
        model = tcn.make_random_tcn(shape, 1, tcn.TCN_WEIGHT_STD[args.net])
        cp = tcn.compile_tcn(shape, be.params)
        be.ensure_rotation_keys(cp.rotations)
        enc = tcn.TcnEncoder(cp, model, be).prepare()
        run = tcn.run_tcn
        encrypt = lambda x: tcn.encrypt_tcn_input(x, cp, be)      # noqa: E731
        decode = lambda out: tcn.dec_tcn_logits(out, enc, be)     # noqa: E731
        clear = lambda x: tcn.infer_clear_tcn(model, x)           # noqa: E731
        desc = f"{args.net} temporal network"
    else:
        shape = net_by_name(args.net)
        cpar = collapse_layers(make_random_model(shape, 1), shape)
        cp = compile_pipeline(shape, "fast", args.strategy, be.params)
        be.ensure_rotation_keys(cp.rotations)
        enc = ModelEncoder(cp, cpar, be).prepare()
        run = None
        encrypt = lambda x: encrypt_input(x, cp, be)              # noqa: E731
        decode = lambda out: dec_logits(out, cp, be)              # noqa: E731
        clear = lambda x: infer_clear(cpar, x)                    # noqa: E731
        desc = f"{args.net} fast/{args.strategy}"
    g1 = GraphedPipeline(enc, be, batch=1, run=run)
    stream = ingest.synthetic_stream(args.frames, shape.joints, seed=7)
    starts = list(range(0, len(stream) - shape.frames + 1, 8))
    lat, srv, agree = [], [], 0
    for k, s in enumerate(starts):
        t0 = time.perf_counter()
        x = ingest.windows(stream[s:s + shape.frames], shape.frames, 8)[0]
        ct = encrypt(x)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        out = g1(ct)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        lg = decode(out)
        t3 = time.perf_counter()
        lat.append((t3 - t0) * 1e3)
        srv.append((t2 - t1) * 1e3)
        if k % 64 == 0:
            agree += int(np.argmax(lg) == np.argmax(clear(x)))
    checked = len(range(0, len(starts), 64))
    # batched throughput over the same windows
    wins = ingest.windows(stream, shape.frames, 8)
    gb = GraphedPipeline(enc, be, batch=args.batch, run=run)
    nb = len(wins) // args.batch
    cts = [encrypt(wins[i * args.batch:(i + 1) * args.batch]) for i in range(nb)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for c in cts:
        gb(c)
    torch.cuda.synchronize()
    thr = nb * args.batch / (time.perf_counter() - t0)
    print(json.dumps({
        "workload": f"streaming {args.frames} frames, 32-frame windows stride 8, "
                    f"{desc}, fast-hear", "windows": len(starts),
        "window_latency_ms": {"p50": float(np.percentile(lat, 50)),
                              "p99": float(np.percentile(lat, 99))},
        "server_eval_latency_ms": {"p50": float(np.percentile(srv, 50)),
                                   "p99": float(np.percentile(srv, 99))},
        "argmax_agreement_vs_clear": f"{agree}/{checked}",
        "batched_windows_per_s": thr, "batch": args.batch}), flush=True)


if __name__ == "__main__":
    main()
