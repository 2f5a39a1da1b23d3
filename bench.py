"""Encrypted HEAR-CNN inference benchmark (B200 engine vs the CPU reference arm).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--net 1d-w64] [--mode fast] [--strategy full] [--batch 128]

One step = one pass of the encrypted network over a batch of B synthetic
clips per GPU (weak scaling: clips are partitioned across ranks, evaluation
keys are generated on rank 0 and broadcast once at setup, no collectives in
the per-clip loop).  Rank 0 prints one JSON line.

  value  encrypted inferences/s over all ranks, inputs already resident in HBM
  e2e    same metric through the public API with host buffers: every step copies
         the encrypted clips host->device (pinned) and the encrypted logits
         device->host
Synthetic data: inputs uniform[0,1) 32x15x2 from seeds, random-init weights of
the named reference network (no datasets or checkpoints on the box).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--net", default="1d-w64")
    ap.add_argument("--mode", default="fast", choices=["fast", "hear"])
    ap.add_argument("--strategy", default="full", choices=["full", "giant", "baby"])
    ap.add_argument("--batch", type=int, default=None,
                    help="clips per GPU per step (default 128); with --workload config2 the "
                         "clips per graph replay (default 64: the N=2^15 graph's temporaries "
                         "at 128 clips plus 4096 resident clips exceed 180 GB)")
    ap.add_argument("--workload", default="default",
                    choices=["default", "config0", "config2", "config3"],
                    help="config2: BASELINE config 2 -- 4096 clips per step at N=2^15 "
                         "(fast-hear ladder), sharded across the ranks (strong scaling); "
                         "config0 / config3: BASELINE's temporal networks (tcn.py) at "
                         "fast-hear (N=2^14) / tcn-2^16")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--check-launch", action="store_true",
                    help="multi-rank plumbing only: spawn, key replication, max-over-ranks")
    args = ap.parse_args()
    if args.batch is None:   # config3: N = 2^16 rows are 4x the default ring's
        args.batch = {"config2": 64, "config3": 32}.get(args.workload, 128)
    return args


def profile_of(mode: str) -> str:
    return "fast-hear" if mode == "fast" else "hear"


def metric_name() -> str:
    return "encrypted HEAR-CNN inferences/sec"


# ---------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        rows = [r for r in self.rows if len(r) >= 7]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


# ---------------------------------------------------------------------------- CPU arm

def workload_params(args):
    from paper_2104_09164_b200.ckks import params as P
    if args.workload == "config2":
        return P.fast_hear_ring(15)
    if args.workload == "config3":
        return P.tcn_ring16()
    return P.gen_params(profile_of(args.mode))


class Workload:
    """One network on one parameter set, behind the calls the harness
    makes: the reference's HEAR networks (compile_pipeline / ModelEncoder /
    run_pipeline) or the temporal networks of BASELINE configs 0 and 3
    (tcn.compile_tcn / TcnEncoder / run_tcn)."""

    def __init__(self, args):
        self.params = workload_params(args)
        self.tcn = args.workload in ("config0", "config3")
        if self.tcn:
            from paper_2104_09164_b200 import tcn
            self.T = tcn
            self.shape = tcn.tcn_by_name(args.workload)
            self.model = tcn.make_random_tcn(self.shape, 1, tcn.TCN_WEIGHT_STD[args.workload])
            self.plan = tcn.compile_tcn(self.shape, self.params)
            self.name = (f"BASELINE {args.workload} temporal network "
                         f"({'; '.join(f'conv k={c.kernel} f={c.filters} s={c.stride}' for c in self.shape.convs)}"
                         f"; {'/'.join(self.shape.acts)}; {self.shape.classes} classes)")
        else:
            from paper_2104_09164_b200.fastpath import compile_pipeline
            from paper_2104_09164_b200.model import collapse_layers, make_random_model
            from paper_2104_09164_b200.model import net_by_name
            self.shape = net_by_name(args.net)
            self.model = collapse_layers(make_random_model(self.shape, 1), self.shape)
            self.plan = compile_pipeline(self.shape, args.mode, args.strategy, self.params)
            self.name = f"HEAR CNN {args.net} {args.mode}/{args.strategy}"

    def encoder(self, be):
        if self.tcn:
            return self.T.TcnEncoder(self.plan, self.model, be).prepare()
        from paper_2104_09164_b200.modelenc import ModelEncoder
        return ModelEncoder(self.plan, self.model, be).prepare()

    @property
    def run(self):
        if self.tcn:
            return self.T.run_tcn
        from paper_2104_09164_b200.fastpath import run_pipeline
        return run_pipeline

    def make_input(self, seed: int):
        if self.tcn:
            return self.T.make_random_clip(self.shape, seed)
        from paper_2104_09164_b200.model import make_random_input
        return make_random_input(self.shape, seed)

    def encrypt(self, x, be):
        if self.tcn:
            return self.T.encrypt_tcn_input(x, self.plan, be)
        from paper_2104_09164_b200.fastpath import encrypt_input
        return encrypt_input(x, self.plan, be)

    def dec(self, out, enc, be):
        if self.tcn:
            return self.T.dec_tcn_logits(out, enc, be)
        from paper_2104_09164_b200.fastpath import dec_logits
        return dec_logits(out, self.plan, be)

    def clear(self, x):
        if self.tcn:
            return self.T.infer_clear_tcn(self.model, x)
        from paper_2104_09164_b200.model import infer_clear
        return infer_clear(self.model, x)


def cpu_oracle_run(args, n_clips: int, warm: int = 0):
    """Time the CPU oracle (oracle/, C + OpenMP port of the reference engine)
    on `n_clips` single-clip inferences.  Returns (clips/s, threads, per-clip s)."""
    from oracle.cpu_engine import OracleCkks, lib
    wl = Workload(args)
    be = OracleCkks(wl.params, seed=0)
    be.ensure_rotation_keys(wl.plan.rotations)
    enc = wl.encoder(be)   # model encoding is setup, not per clip
    cts = [wl.encrypt(wl.make_input(1000 + i), be) for i in range(warm + n_clips)]
    for i in range(warm):
        wl.run(enc, cts[i], be)
    t0 = time.perf_counter()
    for i in range(warm, warm + n_clips):
        wl.run(enc, cts[i], be)
    dt = time.perf_counter() - t0
    return n_clips / dt, int(lib().or_num_threads()), dt / max(n_clips, 1)


def reference_arm(args):
    from paper_2104_09164_b200.parallel import world
    rank, ws, _ = world()
    if rank != 0:
        return
    value, cores, per_clip = cpu_oracle_run(args, args.steps, warm=args.warmup)
    sample = (f"{args.steps} timed single-clip encrypted inferences ({args.warmup} warm-up) of "
              f"{args.net}/{args.mode}/{args.strategy} at {workload_params(args).name} parameters")
    line = {
        "metric": metric_name(), "value": value, "unit": "inferences/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_clip * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": f"{Workload(args).name}, "
                   f"{workload_params(args).name} params, 1 clip per step on the host CPU",
                   "net": args.net, "mode": args.mode, "strategy": args.strategy,
                   "params": workload_params(args).name, "clips_per_step": 1},
        "cpu_baseline": {"value": value, "unit": "inferences/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "inferences/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- GPU arm

FP64_MEASURED_TFLOPS = 17.93   # DFMA/s measured on this pool (profiles/r01_microbench.txt)


TRAFFIC_FILE = os.path.join(ROOT, "profiles", "r2b_roofline_traffic.json")


def dominant_kernel_roofline(be, lvl: int, bsz: int, peaks: dict) -> dict:
    """The kernel with the largest share of the step (step_roofline families,
    profiles/r2b_launches_summary.txt): k_ks3, the fused ModUp + key-switch
    inner product of every non-hoisted key switch.  Engines without it
    (integer-policy rings) report the rotation ModDown as before."""
    if getattr(be, "fuse_ks", False):
        return fused_ks_roofline(be, lvl, bsz, peaks)
    return moddown_roofline(be, lvl, bsz, peaks)


def fused_ks_roofline(be, lvl: int, bsz: int, peaks: dict) -> dict:
    """Time one k_ks3 launch -- the relinearisation key switch of bsz clips at
    level lvl: bsz x (lvl+2) clusters, each the (lvl) forward NTTs of the
    lifted digits under one target prime plus the products with the two key
    rows, sums in tensor memory -- with CUDA events on the launching stream.

    Algorithmic work per launch: bytes = digit coefficient
    rows + their NTT-form identity rows (8N each, once per ciphertext) + the
    key rows (2 x digits x rows, once) + the 2 x rows outputs per ciphertext;
    fp64-pipe instructions = 8 per butterfly of every lift + 6 per modular
    product.  The kernel is bound by the fp64 pipe (its HBM bytes are the
    inputs and outputs only), so `achieved`/`peak` are fp64 instruction rates
    and the HBM side is reported beside them.  `traffic` = DRAM read+write of
    the same launch from an ncu --set full capture (tools/roofline_probe.py)."""
    import torch
    from paper_2104_09164_b200 import _native as nat
    from paper_2104_09164_b200.ckks.engine import _Digits
    from paper_2104_09164_b200.ckks.ring import _upload
    n, logn = be.n, be.n.bit_length() - 1
    ndig, rows = lvl + 1, lvl + 2
    g = torch.Generator(device=be.dev).manual_seed(1)
    src = be.ring.empty(bsz, ndig).random_(0, 1 << 30, generator=g)
    coef = (be.ring.empty(bsz, ndig).random_(0, 1 << 30, generator=g) - (1 << 29)) \
        .to(torch.float64).view(torch.int64)
    ip = be.ring.empty(bsz * 2, rows)
    rp = be.ring.row_ptrs
    key = be.keys.relin
    if key is None:   # a receiver without keys: any resident rows serve as key rows
        raise RuntimeError("roofline probe needs the relinearisation key")
    krow = np.array(list(range(lvl + 1)) + [key.lmax + 1])
    kbr = rp(key.b).reshape(key.b.shape[0], key.lmax + 2)[0, krow]
    kar = rp(key.a).reshape(key.a.shape[0], key.lmax + 2)[0, krow]
    de = _Digits(coef, rp(src).reshape(bsz, ndig), lvl)
    t = be._ksf_tasks(de, lvl, [(kbr, kar, (key.lmax + 2) * n, 0)],
                      rp(ip).reshape(1, bsz, 2, rows), bsz)
    d = _upload(t, be.dev)
    L = nat.lib()
    st = torch.cuda.current_stream()

    def launch():
        nat.check(L.hb_ks_fused(be.ring.handle, d.data_ptr(), len(t), st.cuda_stream), "ks_fused")
    for _ in range(3):
        launch()
    reps = 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(reps):
        launch()
    e1.record(st)
    torch.cuda.synchronize()
    sec = e0.elapsed_time(e1) / 1e3 / reps
    algo = (2 * bsz * ndig + 2 * ndig * rows + 2 * bsz * rows) * 8 * n
    lifts = bsz * (rows * ndig - ndig)
    bfly = lifts * (n // 2) * logn
    fp64_ops = bfly * 8 + 2 * bsz * rows * ndig * n * 6
    gbs = algo / sec / 1e9
    peak_hbm = peaks.get("hbm_gbs", 6650.0)
    fp64_frac = fp64_ops / sec / (FP64_MEASURED_TFLOPS * 1e12)
    traffic = None
    try:
        with open(TRAFFIC_FILE) as f:
            tr = json.load(f)
        if tr.get("kernel") == "k_ks3" and tr.get("tasks") == len(t) and tr.get("n") == n:
            traffic = tr["dram_bytes"]
    except (OSError, ValueError, KeyError):
        pass
    return {"kernel": "k_ks3 (fused ModUp + key-switch inner product, sums in tensor memory)",
            "bound": "fp64", "achieved": round(fp64_ops / sec / 1e12, 3),
            "peak": FP64_MEASURED_TFLOPS, "unit": "T fp64-pipe instr/s",
            "frac": round(fp64_frac, 4), "traffic": traffic, "launch_us": round(sec * 1e6, 2),
            "tasks_per_launch": len(t), "digits": ndig,
            "algorithmic_bytes_per_launch": algo, "fp64_ops_per_launch": fp64_ops,
            "hbm_achieved_gbs": round(gbs, 1), "hbm_peak_gbs": peak_hbm,
            "hbm_frac": round(gbs / peak_hbm, 4),
            "butterflies_per_s": round(bfly / sec / 1e12, 3),
            "peak_source": "fp64: measured DFMA rate on this pool (profiles/r01_microbench.txt); "
                           "hbm: " + ("MEASURED_PEAKS.json" if "hbm_gbs" in peaks else "fallback")}


def moddown_roofline(be, lvl: int, bsz: int, peaks: dict) -> dict:
    """Time one rotation ModDown launch -- k_ntt3_fwd<FWD_MODDOWN_SCATTER>, the
    largest kernel share of the evaluation (profiles/r01_launches_*): the
    ModDown of bsz clips x 2 components x (l+1) rows of a rotation computed on
    pre-permuted keys, result scattered through the inverse Galois map, c0
    added -- with CUDA events on the launching stream.
    Algorithmic bytes: per output row read x_r (8N) + the perm (4N) + write
    (8N); per component-0 row read the addend c0 (8N); per (clip, component)
    one read of the special-prime source row (8N).  `traffic` is the DRAM
    read+write of the same launch from an ncu --set full capture
    (tools/roofline_probe.py -> profiles/r01_roofline_traffic.json)."""
    import torch
    from paper_2104_09164_b200 import _native as nat
    from paper_2104_09164_b200.ckks.engine import _tasks
    from paper_2104_09164_b200.ckks.ring import _upload
    n = be.n
    m, r = bsz * 2, lvl + 1
    g = torch.Generator(device=be.dev).manual_seed(1)
    src = be.ring.empty(m).random_(0, 1 << 30, generator=g)
    lifted = getattr(be, "lift_once", False)
    if lifted:   # the engine's source rows: centred lifts stored as doubles
        src = (src - (1 << 29)).to(torch.float64).view(torch.int64)
    aux = be.ring.empty(m, r).random_(0, 1 << 30, generator=g)
    c0 = be.ring.empty(bsz, r).random_(0, 1 << 30, generator=g)
    out = be.ring.empty(m, r)
    inv = be.ring.perm_inv_for(be.ring.perm_dev(be.ring.galois_element(1)))
    add = np.zeros((bsz, 2, r), dtype=np.uint64)
    add[:, 0] = be.ring.row_ptrs(c0).reshape(bsz, r)
    t = _tasks(nat.NTT_TASK, m * r, src=np.repeat(be.ring.row_ptrs(src), r),
               dst=be.ring.row_ptrs(out), aux=be.ring.row_ptrs(aux),
               src_prime=-1 if lifted else be.S,
               dst_prime=np.tile(np.arange(r), m), scal=np.tile(be._pinv[:r], m),
               scal_sh=np.tile(be._pinv_sh[:r], m), add=add.ravel(),
               perm=np.full(m * r, inv.data_ptr(), dtype=np.uint64))
    d = _upload(t, be.dev)
    L = nat.lib()
    st = torch.cuda.current_stream()

    # two-pass rings (N >= 2^15): the ModDown gathers c0 through the Galois
    # map instead (the scatter form exists on the cluster NTT only)
    mode = nat.FWD_MODDOWN_SCATTER if lifted else nat.FWD_MODDOWN

    def launch():
        nat.check(L.hb_ntt_fwd(be.ring.handle, d.data_ptr(), len(t), mode, st.cuda_stream), "ntt")
    for _ in range(3):
        launch()
    reps = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(reps):
        launch()
    e1.record(st)
    torch.cuda.synchronize()
    sec = e0.elapsed_time(e1) / 1e3 / reps
    # x_r read + output written per row, c0 read per component-0 row, one
    # special-prime source row per (clip, component); the inverse-Galois
    # table is one shared 4N-byte array (L2-resident), counted once
    algo = (m * r * 16 + bsz * r * 8 + m * 8) * n + 4 * n
    gbs = algo / sec / 1e9
    peak = peaks.get("hbm_gbs", 6650.0)
    bfly = m * r * (n // 2) * (n.bit_length() - 1)
    fp64_frac = bfly * 8 / sec / (FP64_MEASURED_TFLOPS * 1e12)
    kname = ("k_ntt3_fwd<FWD_MODDOWN_SCATTER>" if lifted
             else "k_ntt2_cols + k_ntt2_blocks<FWD_MODDOWN> (c0 gathered)")
    traffic = None
    try:
        with open(TRAFFIC_FILE) as f:
            tr = json.load(f)
        if tr.get("kernel") == kname and tr.get("rows") == m * r and tr.get("n") == n:
            traffic = tr["dram_bytes"]
    except (OSError, ValueError, KeyError):
        pass
    # the roof this kernel is nearer to: HBM bytes or the fp64 pipe (its
    # modular butterflies run as fp64 instructions; no tensor-core work)
    hbm_frac = gbs / peak
    bound = "hbm" if hbm_frac >= fp64_frac else "fp64"
    return {"kernel": kname + " (rotation ModDown: NTT + fused epilogue)",
            "bound": bound, "achieved": round(gbs, 1), "peak": peak, "unit": "GB/s",
            "frac": round(hbm_frac, 4), "traffic": traffic, "launch_us": round(sec * 1e6, 2),
            "rows_per_launch": m * r, "algorithmic_bytes_per_launch": algo,
            "butterflies_per_s": round(bfly / sec / 1e12, 3),
            "fp64_frac_of_measured": round(fp64_frac, 3),
            "fp64_peak_ops_per_s": FP64_MEASURED_TFLOPS * 1e12,
            "peak_source": "MEASURED_PEAKS.json" if "hbm_gbs" in peaks else "fallback"}


def step_roofline(enc, ct, be, run_pipeline, ms_graph: float, peaks: dict) -> dict:
    """Step-level roofline: one eager pass of the step with every launch
    accounted (ring.StepStats: algorithmic bytes = distinct source rows once
    + every output row, nominal fp64 instructions of the modular arithmetic)
    and timed with CUDA events around each launch on the launching stream.
    Whole step: the summed algorithmic bytes / fp64 ops over the graph's
    ms_per_step.  Per kernel family: its share of the eager step's device
    time, achieved GB/s and fp64 fraction over its own launches."""
    import torch
    from paper_2104_09164_b200.ckks import ring as R
    peak = peaks.get("hbm_gbs", 6650.0)
    fp64_peak = FP64_MEASURED_TFLOPS * 1e12
    st = R.StepStats(timed=True)
    R.set_step_stats(st)
    try:
        torch.cuda.synchronize()
        run_pipeline(enc, ct, be)
        fam = st.finish()
    finally:
        R.set_step_stats(None)
    tot_b = sum(f["bytes"] for f in fam.values())
    tot_f = sum(f["fp64_ops"] for f in fam.values())
    tot_ms = sum(f["ms"] for f in fam.values())
    fams = {}
    for name, f in sorted(fam.items(), key=lambda kv: -kv[1]["ms"]):
        sec = max(f["ms"], 1e-9) / 1e3
        fams[name] = {"launches": f["launches"], "share": round(f["ms"] / tot_ms, 4),
                      "ms": round(f["ms"], 3), "algorithmic_bytes": f["bytes"],
                      "achieved_gbs": round(f["bytes"] / sec / 1e9, 1),
                      "hbm_frac": round(f["bytes"] / sec / 1e9 / peak, 4),
                      "fp64_frac": round(f["fp64_ops"] / sec / fp64_peak, 4)}
    sec = ms_graph / 1e3
    return {"algorithmic_bytes_per_step": tot_b, "fp64_ops_per_step": tot_f,
            "hbm_frac": round(tot_b / sec / 1e9 / peak, 4),
            "fp64_frac": round(tot_f / sec / fp64_peak, 4),
            "eager_step_device_ms": round(tot_ms, 3), "graph_ms_per_step": round(ms_graph, 3),
            "fp64_ops_note": "8 per NTT butterfly, 6 per modular product (fmod_mul + accumulate), "
                             "3 per product of the split-sum layer MAC",
            "families": fams}


def keyswitch_rate(be, lvl: int, bsz: int) -> dict:
    """Key-switch ops/s at level lvl on one handle of bsz clips: HRotate by
    one amount (bsz key switches: ModUp + inner product + ModDown +
    automorphism) and the hoisted form (16 amounts sharing the ModUp).
    Eager calls timed with CUDA events, best of 3 blocks of 3 calls."""
    import torch
    from fractions import Fraction
    from paper_2104_09164_b200.backend import Ct
    from paper_2104_09164_b200.ckks.engine import CtData
    be.ensure_rotation_keys({k: be.L for k in range(1, 17)})
    big = Ct(CtData(be.ring.empty(bsz, 2, lvl + 1).random_(0, 1 << 30)), lvl, Fraction(1), be.n2)
    out = {}
    for name, fn, ops in (("rotate", lambda: be._raw_rot(big, 1), bsz),
                          ("rotate_hoisted16",
                           lambda: be._raw_rot_many(big, list(range(1, 17))), 16 * bsz)):
        fn()
        torch.cuda.synchronize()
        best = 0.0
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                fn()
            e1.record()
            torch.cuda.synchronize()
            best = max(best, 3 * ops / (e0.elapsed_time(e1) / 1e3))
        out[name] = round(best, 1)
    out["level"] = lvl
    out["clips"] = bsz
    out["unit"] = "key-switch ops/s"
    return out


def gpu_arm(args):
    import torch
    from paper_2104_09164_b200 import _native as nat
    from paper_2104_09164_b200 import parallel as par
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params
    from paper_2104_09164_b200.backend import Ct
    from paper_2104_09164_b200.ckks.engine import CtData
    from paper_2104_09164_b200.fastpath import GraphedPipeline

    rank, ws, local = par.world()
    if ws != args.gpus:
        raise SystemExit(f"world size {ws} != --gpus {args.gpus}: launch with torchrun "
                         "or let bench.py spawn the ranks")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    par.init("nccl")
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass

    if args.workload == "config2" and args.mode != "fast":
        raise SystemExit("config2 runs the fast-hear ladder (--mode fast)")
    wl = Workload(args)
    params = wl.params
    run_pipeline = wl.run
    # receivers encrypt from their own stream (never the sender's keygen stream)
    be = CkksBackend(params, seed=0, device=dev, keygen=(rank == 0),
                     enc_seed=np.random.SeedSequence(0, spawn_key=(rank,)))
    if rank == 0:
        be.ensure_rotation_keys(wl.plan.rotations)
    par.replicate_keys(be, src=0)
    enc = wl.encoder(be)
    if args.workload == "config2":
        # 4096 clips per step over all ranks, each rank's shard resident in
        # HBM as handles of `batch` clips (one graph replay each)
        mine = list(par.shard(4096, rank, ws))
        bsz = min(args.batch, len(mine))
        if len(mine) % bsz:
            raise SystemExit(f"{len(mine)} clips per rank is not a multiple of --batch {bsz}")
        seeds = [10_000 + i for i in mine]
    else:
        bsz = args.batch
        seeds = [10_000 * (rank + 1) + i for i in range(bsz)]
    chunks, xs = [], []
    for c0 in range(0, len(seeds), bsz):
        xc = np.stack([wl.make_input(s) for s in seeds[c0:c0 + bsz]])
        chunks.append(wl.encrypt(xc, be))
        xs.append(xc)
    ct, x = chunks[0], xs[0]
    host_in = [c.payload.data.cpu().pin_memory() for c in chunks]
    out0 = run_pipeline(enc, ct, be)
    host_out = [torch.empty(out0.payload.data.shape, dtype=torch.int64).pin_memory()
                for _ in chunks]
    torch.cuda.synchronize()
    maxerr = None
    if rank == 0:
        lg = wl.dec(out0, enc, be)
        ref = np.stack([wl.clear(xi) for xi in x])
        maxerr = float(np.abs(lg - ref).max())

    st = torch.cuda.current_stream()
    # kernels per step, counted by the library on an eager pass
    k0 = nat.kernel_launches()
    run_pipeline(enc, ct, be)
    per_step_kernels = nat.kernel_launches() - k0
    # the timed loops replay the pipeline captured as one CUDA graph
    graph = GraphedPipeline(enc, be, batch=bsz, run=wl.run)
    for _ in range(args.warmup):
        graph(ct)
    torch.cuda.synchronize()

    # ---- device-resident timed region
    par.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    prof_range = os.environ.get("HEAR_PROFILE_RANGE") == "1"  # ncu --profile-from-start off
    with ClockSampler(local) as clk:
        if prof_range:
            torch.cuda.profiler.start()
        e0.record(st)
        for _ in range(args.steps):
            for c in chunks:
                graph(c)
        e1.record(st)
        torch.cuda.synchronize()
        if prof_range:
            torch.cuda.profiler.stop()
    launches = per_step_kernels * args.steps * len(chunks)
    par.barrier()
    ms = par.max_over_ranks(e0.elapsed_time(e1) / args.steps, dev)

    # ---- end-to-end timed region (host buffers, copies inside).  Every step
    # copies its input from pinned host memory and reads its result back;
    # the copies run on a side stream double-buffered against the replays
    # (step s+1's H2D and step s-1's D2H overlap step s's evaluation)
    par.barrier()
    torch.cuda.synchronize()
    cs = torch.cuda.Stream(device=dev)
    stage_in = [torch.empty_like(graph.inp) for _ in range(2)]
    stage_out = [torch.empty_like(graph.out.payload.data) for _ in range(2)]
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_free = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    ev_d2h = [torch.cuda.Event() for _ in range(2)]
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nch = len(chunks)
    jobs = args.steps * nch    # one job = one handle of bsz clips (a graph replay)
    f0.record(st)
    cs.wait_stream(st)
    with torch.cuda.stream(cs):
        stage_in[0].copy_(host_in[0], non_blocking=True)
        ev_in[0].record(cs)
    for i in range(jobs):
        b = i % 2
        st.wait_event(ev_in[b])
        graph.inp.copy_(stage_in[b])
        ev_free[b].record(st)
        if i + 1 < jobs:   # next job's input, into the other staging buffer
            with torch.cuda.stream(cs):
                if i >= 1:
                    cs.wait_event(ev_free[1 - b])
                stage_in[1 - b].copy_(host_in[(i + 1) % nch], non_blocking=True)
                ev_in[1 - b].record(cs)
        graph.graph.replay()
        if i >= 2:   # job i-2's read-back of this staging buffer is done
            st.wait_event(ev_d2h[b])
        stage_out[b].copy_(graph.out.payload.data)
        ev_out[b].record(st)
        with torch.cuda.stream(cs):
            cs.wait_event(ev_out[b])
            host_out[i % nch].copy_(stage_out[b], non_blocking=True)
            ev_d2h[b].record(cs)
    st.wait_stream(cs)
    f1.record(st)
    torch.cuda.synchronize()
    par.barrier()
    ms_e2e = par.max_over_ranks(f0.elapsed_time(f1) / args.steps, dev)
    if rank == 0:   # the replays' outputs decrypt to the clear network's logits
        for q in sorted({0, nch - 1}):
            fc = wl.plan.expected("fc")
            out_ct = Ct(CtData(host_out[q].to(dev)), fc.level, fc.scale, be.n2)
            refq = np.stack([wl.clear(xi) for xi in xs[q]])
            maxerr = max(maxerr, float(np.abs(wl.dec(out_ct, enc, be) - refq).max()))

    # ---- per-clip latency: single-clip graph, replays timed one by one
    lat = []
    g1 = GraphedPipeline(enc, be, batch=1, run=wl.run)
    one = wl.encrypt(x[0], be)
    for i in range(3 + max(args.steps, 10)):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        g1(one)
        b.record(st)
        torch.cuda.synchronize()
        if i >= 3:
            lat.append(a.elapsed_time(b))
    latency = {"p50_ms": float(np.percentile(lat, 50)), "p99_ms": float(np.percentile(lat, 99)),
               "samples": len(lat), "batch": 1}
    del g1, graph

    roof = ks = steproof = None
    if rank == 0:
        steproof = step_roofline(enc, ct, be, run_pipeline, ms / len(chunks), peaks)
    if rank == 0:   # per-GPU kernel figures; the other ranks hold no secret key
        # one rotation ModDown over 64 clips (the shape of the committed ncu capture)
        roof = dominant_kernel_roofline(be, lvl=params.max_level, bsz=64, peaks=peaks)
        ks = keyswitch_rate(be, lvl=params.max_level, bsz=min(bsz, 32))

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            v, cores, per_clip = cpu_oracle_run(args, 1)
            cpu = {"value": v, "unit": "inferences/s", "cores": cores, "kind": "port",
                   "sample": f"1 single-clip encrypted inference of {args.net}/{args.mode}/"
                             f"{args.strategy} ({per_clip:.1f} s) on the oracle C/OpenMP port"}
        except Exception as exc:  # the oracle must not break the GPU number
            cpu = {"value": None, "unit": "inferences/s", "cores": os.cpu_count(),
                   "kind": "port", "sample": f"failed: {exc}"}

    if rank == 0 and not maxerr <= 2.0 ** -5:
        # the documented precision of the encrypted network vs the clear one
        # (DESIGN.md §2); a larger error means a broken kernel: no number
        raise SystemExit(f"decrypted logits deviate from the clear network by {maxerr}")
    if rank == 0:
        per_gpu = bsz * len(chunks)
        total = per_gpu * ws
        per_step = (f"BASELINE config 2: 4096 clips per step sharded over {ws} GPU(s), "
                    f"{len(chunks)} handles of {bsz} clips per GPU" if args.workload == "config2"
                    else f"{bsz} clips per GPU per step")
        line = {
            "metric": metric_name(), "value": total / (ms / 1e3), "unit": "inferences/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "strong" if args.workload == "config2" else "weak",
            "vs_baseline": None, "dtype": "u64",
            "data": "synthetic",
            "config": {"workload": f"{wl.name}, "
                       f"{params.name} params (N=2^{params.n.bit_length() - 1}, L={params.max_level}),"
                       f" {per_step}", "net": args.net if not wl.tcn else args.workload,
                       "mode": args.mode,
                       "strategy": args.strategy, "params": params.name, "clips_per_gpu": per_gpu,
                       "clips_per_replay": bsz,
                       "global_clips_per_step": total, "parallelism": f"clip-sharded dp{ws}",
                       "l2": "working set (keys + plaintexts + ciphertexts) >> 126 MB L2",
                       "latency_ms_per_batch": ms, "decrypt_max_abs_err_vs_clear": maxerr},
            "e2e": {"value": total / (ms_e2e / 1e3), "unit": "inferences/s",
                    "h2d_bytes_per_step": int(sum(h.numel() for h in host_in) * 8),
                    "d2h_bytes_per_step": int(sum(h.numel() for h in host_out) * 8)},
            "gpu_launches": launches,
            "per_clip_latency": latency,
            "keyswitch": ks,
            "roofline": roof,
            "step_roofline": steproof,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    par.barrier()


def launch_check(args):
    """The multi-rank path without the encrypted network: world size, the
    setup-time key broadcast over tensors of the real key layout (toy-fast
    parameters, the toy network's rotation manifest), max over ranks.  Runs
    on CPU (gloo) as well as on GPUs (NCCL)."""
    import torch
    import torch.distributed as dist
    from paper_2104_09164_b200 import parallel as par
    from paper_2104_09164_b200.ckks.engine import key_layout
    from paper_2104_09164_b200.ckks.params import gen_params
    from paper_2104_09164_b200.fastpath import compile_pipeline
    from paper_2104_09164_b200.model import NetworkShape
    rank, ws, local = par.world()
    cuda = torch.cuda.is_available()
    dev = torch.device("cuda", local) if cuda else torch.device("cpu")
    if cuda:
        torch.cuda.set_device(local)
    par.init("nccl" if cuda else "gloo")
    if ws != args.gpus:
        raise SystemExit(f"world size {ws} != --gpus {args.gpus}")
    ps = gen_params("toy-fast")
    cp = compile_pipeline(NetworkShape(1, 32, 15, (4, 8, 16), 4), "fast", "giant", ps)
    manifest = par.broadcast_object(sorted(cp.rotations.items()) if rank == 0 else None)
    layout = key_layout(ps, manifest)
    g = torch.Generator().manual_seed(7)
    keys = [torch.randint(0, 1 << 40, shape, generator=g).to(dev) if rank == 0 else
            torch.empty(shape, dtype=torch.int64, device=dev) for _, shape in layout]
    par.broadcast_tensors(keys)
    sums = torch.tensor([float(sum(int(k.sum()) for k in keys) % (1 << 50))], dtype=torch.float64,
                        device=dev)
    allsum = [torch.zeros_like(sums) for _ in range(ws)] if ws > 1 else [sums]
    if ws > 1:
        dist.all_gather(allsum, sums)
    mx = par.max_over_ranks(float(rank + 1), dev)
    if rank == 0:
        print(json.dumps({"check": "launch", "n_ranks": ws, "backend": "nccl" if cuda else "gloo",
                          "key_tensors": len(keys),
                          "key_bytes": int(sum(k.numel() * 8 for k in keys)),
                          "keys_identical": len({float(t.item()) for t in allsum}) == 1,
                          "max_over_ranks": mx}), flush=True)
    par.barrier()


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` started as one process: become N ranks
        from paper_2104_09164_b200.parallel import relaunch
        sys.exit(relaunch(args.gpus, os.path.abspath(__file__), sys.argv[1:]))
    if args.check_launch:
        launch_check(args)
    elif args.impl == "reference":
        reference_arm(args)
    else:
        gpu_arm(args)


if __name__ == "__main__":
    main()
