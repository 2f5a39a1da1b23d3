"""Ring context: NTT twiddle tables, Galois permutations and the device-side
launch helpers over RNS row polynomials.

Host-side tables are exact Python-integer computations of the same values
hear/ckks/ring.py:253-364 builds (bit-reversed psi powers per prime, the NTT
evaluation-exponent map, NTT-domain Galois permutations).  One deliberate
difference: the inverse table holds psi^-brv(j), the true inverse of the
forward transform; the reference's table (ring.py:282, exponent brv(j)+1)
makes intt(ntt(a)) != a, so its decryptions are garbage.

All polynomial data lives on the GPU as int64 torch tensors reinterpreted as
uint64 by the kernels; a "row" is N contiguous residues under one prime.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from .. import _native as nat
from .ntheory import bit_reverse_table, root_2n


class UploadArena:
    """Persistent device buffer for task tables while a CUDA graph is being
    captured: every table gets its own never-reused slice, written once at
    capture time through a side stream (the capture runs in relaxed mode),
    so replays read the tables in place and the graph carries no
    host-to-device copy nodes.  Sized before the capture from a counted
    eager pass (no allocation inside the capture)."""

    def __init__(self, device, nbytes: int = 256 << 20):
        self.host = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
        self.dev = torch.empty(nbytes, dtype=torch.uint8, device=device)
        self.off = 0
        self.side = torch.cuda.Stream(device)

    def put(self, t: torch.Tensor) -> torch.Tensor:
        n = t.numel()
        start = (self.off + 255) & ~255
        if start + n > self.dev.numel():
            raise MemoryError("graph upload arena exhausted")
        self.host[start:start + n].copy_(t)
        d = self.dev[start:start + n]
        with torch.cuda.stream(self.side):
            d.copy_(self.host[start:start + n], non_blocking=True)
        self.side.synchronize()
        self.off = start + n
        return d


class UploadCounter:
    """Counts the arena bytes (256-B aligned) an eager pass uploads."""

    def __init__(self):
        self.nbytes = 0

    def add(self, n: int):
        self.nbytes += (n + 255) & ~255


_ARENA: UploadArena | None = None
_COUNTER: UploadCounter | None = None


def set_upload_arena(arena: UploadArena | None):
    global _ARENA
    _ARENA = arena


def set_upload_counter(counter: UploadCounter | None):
    global _COUNTER
    _COUNTER = counter


def _upload(arr: np.ndarray, device) -> torch.Tensor:
    """Host task table -> device bytes (async on the current stream)."""
    t = torch.from_numpy(np.ascontiguousarray(arr).view(np.uint8))
    if t.numel() == 0:
        return torch.empty(0, dtype=torch.uint8, device=device)
    if _COUNTER is not None:
        _COUNTER.add(t.numel())
    if _ARENA is not None:
        return _ARENA.put(t)
    return t.pin_memory().to(device, non_blocking=True)


def _ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


class StepStats:
    """Algorithmic accounting of every launch helper below, for the step-level
    roofline in bench.py: per kernel family, the launches, the ALGORITHMIC
    HBM bytes (each distinct source row counted once per launch, every
    destination row once; shared tables such as Galois permutations and
    twiddles once per launch) and the modular products; with `timed`, also
    the device time of each launch (CUDA events around it on the launching
    stream, resolved by `finish`).  Enabled with `set_step_stats`; the
    launch helpers do no accounting otherwise."""

    FP64_PER_BUTTERFLY = 8   # fmod_mul (5) + add + sub + conditional correction
    FP64_PER_MODMUL = 6      # fmod_mul (5) + accumulate
    FP64_PER_SPLITMUL = 3    # mac.cu split sums: 2 DFMA + operand conversions / reductions

    def __init__(self, timed: bool = False):
        self.timed = timed
        self.fam: dict = {}
        self._ev: list = []

    def add(self, fam: str, nbytes: int, fp64: int, kernels: int = 1):
        r = self.fam.setdefault(fam, {"launches": 0, "bytes": 0, "fp64_ops": 0, "ms": 0.0})
        r["launches"] += kernels
        r["bytes"] += int(nbytes)
        r["fp64_ops"] += int(fp64)

    def begin(self):
        if not self.timed:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    def end(self, fam: str, e0):
        if e0 is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record()
            self._ev.append((fam, e0, e1))

    def finish(self):
        torch.cuda.synchronize()
        for fam, e0, e1 in self._ev:
            self.fam[fam]["ms"] += e0.elapsed_time(e1)
        self._ev = []
        return self.fam


_STATS: StepStats | None = None


def set_step_stats(stats: StepStats | None):
    global _STATS
    _STATS = stats


def _uniq(col) -> int:
    col = np.asarray(col, dtype=np.uint64).ravel()
    return int(np.count_nonzero(np.unique(col)))


class RingContext:
    """Per-parameter-set tables (host) and the kernel library handle (device).

    Global prime index: chain primes 0..L, then the special prime (L+1)."""

    def __init__(self, params, device=None):
        self.params = params
        self.n = params.n
        self.logn = self.n.bit_length() - 1
        self.primes = list(params.chain_primes) + [params.special_prime]
        self.special_idx = len(self.primes) - 1
        self.device = torch.device(device or "cuda")
        if self.device.type != "cuda" or not torch.cuda.is_available():
            raise nat.NativeError("the B200 engine needs a CUDA device (no CPU fallback)")
        self.p = np.array(self.primes, dtype=np.uint64)
        n, logn = self.n, self.logn
        brv = bit_reverse_table(logn)
        self.psi = np.zeros((len(self.primes), n), dtype=np.uint64)
        self.ipsi = np.zeros((len(self.primes), n), dtype=np.uint64)
        for i, q in enumerate(self.primes):
            root = root_2n(q, 2 * n)
            self.psi[i] = _powers(root, brv, q)
            self.ipsi[i] = _powers(pow(root, -1, q), brv, q)
        # NTT output j evaluates at psi^(2 brv(j) + 1) (probed in ring.py:320-334)
        self.exp_map = 2 * brv + 1
        self._perm_host: dict = {}
        self._perm_dev: dict = {}
        L = nat.lib()
        h = L.hb_ring_create(logn, len(self.primes), self.p.ctypes.data,
                             self.psi.ctypes.data, self.ipsi.ctypes.data)
        if not h:
            raise nat.NativeError(L.hb_last_error().decode())
        self.handle = ctypes.c_void_p(h)
        self._lib = L

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self._lib.hb_ring_destroy(self.handle)
        except Exception:
            pass

    # ---- Galois machinery (ring.py:336-364) --------------------------------

    def galois_element(self, r: int) -> int:
        """X -> X^g realising a left slot rotation by r."""
        return pow(5, r % (self.n // 2), 2 * self.n)

    def ntt_perm(self, g: int) -> np.ndarray:
        """out[j] = in[perm[j]] applies X -> X^g to NTT-domain rows."""
        if g not in self._perm_host:
            two_n = 2 * self.n
            pos = np.full(two_n, -1, dtype=np.int64)
            pos[self.exp_map] = np.arange(self.n)
            perm = pos[(self.exp_map * g) % two_n]
            if perm.min() < 0:
                raise RuntimeError("automorphism leaves the evaluation set")
            self._perm_host[g] = perm.astype(np.int32)
        return self._perm_host[g]

    def perm_dev(self, g: int) -> torch.Tensor:
        if g not in self._perm_dev:
            self._perm_dev[g] = torch.from_numpy(self.ntt_perm(g)).to(self.device)
        return self._perm_dev[g]

    def perm_inv_dev(self, g: int) -> torch.Tensor:
        """Inverse of ntt_perm(g) (scatter index of a pre-permuted rotation)."""
        key = -g
        if key not in self._perm_dev:
            perm = self.ntt_perm(g)
            inv = np.empty_like(perm)
            inv[perm] = np.arange(len(perm), dtype=perm.dtype)
            self._perm_dev[key] = torch.from_numpy(inv).to(self.device)
            self._perm_dev[("inv", self.perm_dev(g).data_ptr())] = self._perm_dev[key]
        return self._perm_dev[key]

    def perm_inv_for(self, perm: torch.Tensor) -> torch.Tensor:
        """Inverse permutation of a tensor returned by perm_dev."""
        hit = self._perm_dev.get(("inv", perm.data_ptr()))
        if hit is None:
            for g, t in list(self._perm_dev.items()):
                if isinstance(g, int) and g > 0 and t.data_ptr() == perm.data_ptr():
                    return self.perm_inv_dev(g)
            raise KeyError("unknown permutation")
        return hit

    def coeff_automorphism(self, coeffs: np.ndarray, g: int) -> np.ndarray:
        """X -> X^g on signed integer coefficients."""
        k = np.arange(self.n, dtype=np.int64)
        e = (k * g) % (2 * self.n)
        out = np.zeros_like(coeffs)
        out[e % self.n] = np.where(e >= self.n, -coeffs, coeffs)
        return out

    # ---- launch helpers ------------------------------------------------------

    @property
    def stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def _ntt_kernels(self, count: int) -> int:
        """Kernels one NTT call enqueues (csrc/ntt.cu ntt_kernels)."""
        return int(self._lib.hb_ntt_kernels(self.handle, count))

    _FWD_NAMES = {nat.FWD_PLAIN: "ntt_fwd", nat.FWD_LIFT: "ntt_fwd_modup_lift",
                  nat.FWD_MODDOWN: "ntt_fwd_moddown", nat.FWD_I64: "ntt_fwd_i64",
                  nat.FWD_MODDOWN_SCATTER: "ntt_fwd_moddown_scatter",
                  nat.FWD_MODDOWN2: "ntt_fwd_moddown_rescale"}

    def _ntt_account(self, fam: str, tasks: np.ndarray, kernels: int):
        row = 8 * self.n
        m = len(tasks)
        nbytes = (_uniq(tasks["src"]) + m) * row             # sources once, every output
        if fam == "ntt_fwd_moddown_rescale":   # perm = second source row, add2 = a scalar
            nbytes += (_uniq(tasks["aux"]) + _uniq(tasks["add"]) + _uniq(tasks["perm"])) * row
            nbytes += m * 16 * self.n // 8
        else:
            nbytes += (_uniq(tasks["aux"]) + _uniq(tasks["add"]) + _uniq(tasks["add2"])) * row
            nbytes += _uniq(tasks["perm"]) * 4 * self.n + m * 16 * self.n // 8   # perms; twiddles
        fp64 = m * (self.n // 2) * self.logn * StepStats.FP64_PER_BUTTERFLY
        if fam.startswith("ntt_fwd_moddown"):
            fp64 += m * self.n * StepStats.FP64_PER_MODMUL
        _STATS.add(fam, nbytes, fp64, kernels)

    def ntt_fwd(self, tasks: np.ndarray, mode: int = nat.FWD_PLAIN):
        if len(tasks):
            d = _upload(tasks, self.device)
            k = self._ntt_kernels(len(tasks))
            fam = self._FWD_NAMES.get(mode, "ntt_fwd")
            e0 = _STATS.begin() if _STATS else None
            nat.check(self._lib.hb_ntt_fwd(self.handle, _ptr(d), len(tasks), mode, self.stream),
                      "ntt_fwd", k)
            if _STATS:
                _STATS.end(fam, e0)
                self._ntt_account(fam, tasks, k)

    def ntt_inv(self, tasks: np.ndarray):
        if len(tasks):
            d = _upload(tasks, self.device)
            k = self._ntt_kernels(len(tasks))
            e0 = _STATS.begin() if _STATS else None
            nat.check(self._lib.hb_ntt_inv(self.handle, _ptr(d), len(tasks), self.stream),
                      "ntt_inv", k)
            if _STATS:
                _STATS.end("ntt_inv", e0)
                self._ntt_account("ntt_inv", tasks, k)

    _EW_READS = {nat.EW_ADD: ("a", "b"), nat.EW_SUB: ("a", "b"), nat.EW_MUL: ("a", "b"),
                 nat.EW_MUL_SCALAR: ("a",), nat.EW_MULADD: ("a", "b", "c"),
                 nat.EW_ADD_SCALED: ("a", "b"), nat.EW_COPY: ("a",), nat.EW_PERM: ("a",),
                 nat.EW_SUB_SCALED: ("a", "b"), nat.EW_PERM_ADD: ("a", "b"),
                 nat.EW_MD_TOP: ("a", "b", "c")}
    _EW_MULS = {nat.EW_MUL: 1, nat.EW_MUL_SCALAR: 1, nat.EW_MULADD: 1, nat.EW_ADD_SCALED: 1,
                nat.EW_SUB_SCALED: 1}

    def ew(self, op: int, tasks: np.ndarray):
        if len(tasks):
            d = _upload(tasks, self.device)
            e0 = _STATS.begin() if _STATS else None
            nat.check(self._lib.hb_ew(self.handle, op, _ptr(d), len(tasks), self.stream), "ew")
            if _STATS:
                _STATS.end("elementwise", e0)
                rd = self._EW_READS.get(op, ())
                rows = (_uniq(np.concatenate([tasks[f] for f in rd])) if rd else 0) + len(tasks)
                nbytes = rows * 8 * self.n
                if op == nat.EW_PERM:
                    nbytes += _uniq(tasks["b"]) * 4 * self.n
                if op == nat.EW_PERM_ADD:
                    nbytes += _uniq(tasks["c"]) * 4 * self.n
                _STATS.add("elementwise", nbytes,
                           len(tasks) * self.n * self._EW_MULS.get(op, 0) * StepStats.FP64_PER_MODMUL)

    def mac_strided(self, outs: np.ndarray, terms: np.ndarray, rows: int, bc: int):
        if len(outs):
            d, t = _upload(outs, self.device), _upload(terms, self.device)
            e0 = _STATS.begin() if _STATS else None
            nat.check(self._lib.hb_mac_strided(self.handle, _ptr(d), len(outs), _ptr(t), rows, bc,
                                               self.stream), "mac_strided")
            if _STATS:
                _STATS.end("mac_strided", e0)
                row = 8 * self.n
                nbytes = (_uniq(terms["pt"]) * rows + _uniq(terms["ct"]) * rows * bc
                          + len(outs) * rows * bc) * row
                _STATS.add("mac_strided", nbytes,
                           len(terms) * rows * bc * self.n * StepStats.FP64_PER_MODMUL)

    def sum_rows(self, dst: np.ndarray, srcs: np.ndarray, primes: np.ndarray):
        """dst[r] = sum_k srcs[r, k] (mod p_r) for every output row r."""
        rows, k = srcs.shape
        if rows:
            tasks = np.zeros(rows, dtype=nat.MAC_TASK)
            tasks["dst"], tasks["prime"] = dst, primes
            tasks["nterms"], tasks["term_off"] = k, np.arange(rows) * k
            d = _upload(tasks, self.device)
            s = _upload(np.ascontiguousarray(srcs, dtype=np.uint64).ravel(), self.device)
            e0 = _STATS.begin() if _STATS else None
            nat.check(self._lib.hb_sum(self.handle, _ptr(d), rows, _ptr(s), self.stream), "sum")
            if _STATS:
                _STATS.end("sum_rows", e0)
                _STATS.add("sum_rows", (_uniq(srcs) + rows) * 8 * self.n, 0)

    def tensor(self, tasks: np.ndarray):
        if len(tasks):
            d = _upload(tasks, self.device)
            e0 = _STATS.begin() if _STATS else None
            nat.check(self._lib.hb_tensor(self.handle, _ptr(d), len(tasks), self.stream),
                      "tensor")
            if _STATS:
                _STATS.end("tensor", e0)
                rd = _uniq(np.concatenate([tasks[f] for f in ("a0", "a1", "b0", "b1")]))
                _STATS.add("tensor", (rd + 3 * len(tasks)) * 8 * self.n,
                           4 * len(tasks) * self.n * StepStats.FP64_PER_MODMUL)

    def mac_shared(self, cts: np.ndarray, pts: np.ndarray, dsts: np.ndarray, rows: int, bc: int,
                   pts_last: np.ndarray | None = None, prime_last: int = 0):
        """Shared-term MAC: dsts[o] = sum_t pts[o, t] * cts[t] over [bc, rows, N] blocks.
        pts_last: extended-basis blocks -- the last row is the special prime's,
        its plaintext rows given by pointer ([nout, nterms])."""
        nout, nterms = pts.shape
        if nout:
            parts = [cts.ravel(), pts.ravel(), dsts.ravel()]
            if pts_last is not None:
                parts.append(pts_last.ravel())
            buf = _upload(np.concatenate(parts).astype(np.uint64), self.device)
            base = _ptr(buf)
            o_pts, o_dst = base + 8 * nterms, base + 8 * (nterms + nout * nterms)
            e0 = _STATS.begin() if _STATS else None
            if pts_last is None:
                nat.check(self._lib.hb_mac_shared(self.handle, base, o_pts, o_dst, nterms, nout,
                                                  rows, bc, self.stream), "mac_shared")
            else:
                nat.check(self._lib.hb_mac_shared_ext(self.handle, base, o_pts, o_dst + 8 * nout,
                                                      o_dst, nterms, nout, rows, bc, prime_last,
                                                      self.stream), "mac_shared_ext")
            if _STATS:   # ct terms [bc, rows, N] once, pt rows once, outputs
                _STATS.end("layer_mac_gemm", e0)
                nbytes = (_uniq(cts) * bc + _uniq(pts) + nout * bc) * rows * 8 * self.n
                # long term lists on small primes take the split partial sums:
                # 2 DFMA per product + conversions and periodic reductions
                per = StepStats.FP64_PER_SPLITMUL if (nterms > 32 and nout > 4 and self.split_ok) \
                    else StepStats.FP64_PER_MODMUL
                _STATS.add("layer_mac_gemm", nbytes, nout * nterms * bc * rows * self.n * per)

    @property
    def split_ok(self) -> bool:
        """mac.cu sums split products exactly (every prime below 2^34)."""
        return (self.use_f64 and max(self.primes) < (1 << 34)
                and os.environ.get("HEAR_B200_MAC_SPLIT", "1") != "0")

    @property
    def use_f64(self) -> bool:
        """Modular arithmetic on the fp64 pipe (csrc/cabi.cu policy)."""
        return bool(self._lib.hb_ring_uses_f64(self.handle))

    def ks_gemm(self, de: np.ndarray, keys: np.ndarray, keys_last: np.ndarray, dsts: np.ndarray,
                rows: int, bc: int, de_bstride: int, dst_bstride: int, prime_last: int,
                rot=None):
        """Natural-order key-switch inner products as one per-coefficient GEMM
        (csrc/mac.cu launch_ks_gemm): de [ndig] shared or [njobs, ndig] per job,
        keys / keys_last [nout, ndig], dsts [nout].  rot = (scat [nout], c0s
        [nout], c0_bstride, pmod device pointer): the rotation epilogue
        (hb_ks_gemm_rot) -- outputs scattered through scat[o] with P * c0 added
        on the chain rows, i.e. rotated ciphertexts in the extended basis."""
        nout, ndig = keys.shape
        if nout:
            per_job = int(de.ndim == 2)
            parts = [de.ravel(), keys.ravel(), keys_last.ravel(), dsts.ravel()]
            if rot is not None:
                parts += [np.asarray(rot[0], dtype=np.uint64), np.asarray(rot[1], dtype=np.uint64)]
            buf = _upload(np.concatenate(parts).astype(np.uint64), self.device)
            base = _ptr(buf)
            o1 = base + 8 * de.size
            o2 = o1 + 8 * keys.size
            o3 = o2 + 8 * keys.size
            e0 = _STATS.begin() if _STATS else None
            if rot is None:
                nat.check(self._lib.hb_ks_gemm(self.handle, base, o1, o2, o3, ndig, nout, rows, bc,
                                               de_bstride, dst_bstride, prime_last, per_job,
                                               self.stream), "ks_gemm")
            else:
                o4 = o3 + 8 * nout
                c0 = int(max(rot[1]))
                nat.check(self._lib.hb_ks_gemm_rot(self.handle, base, o1, o2, o3, o4, o4 + 8 * nout,
                                                   c0, rot[3], ndig, nout, rows, bc, de_bstride,
                                                   dst_bstride, rot[2], prime_last, self.stream),
                          "ks_gemm_rot")
            if _STATS:   # digit sets [bc, ndig, rows] once, key rows once, outputs
                _STATS.end("keyswitch_gemm", e0)
                nbytes = (_uniq(de) * bc * rows + _uniq(keys) * (rows - 1) + _uniq(keys_last)
                          + nout * bc * rows) * 8 * self.n
                if rot is not None:   # c0 rows once per clip, scatter maps once
                    nbytes += _uniq(rot[1]) * bc * (rows - 1) * 8 * self.n + _uniq(rot[0]) * 4 * self.n
                _STATS.add("keyswitch_gemm", nbytes, nout * ndig * bc * rows * self.n
                           * StepStats.FP64_PER_MODMUL)

    def ks_fused(self, tasks: np.ndarray):
        """Fused ModUp + key-switch inner product (csrc/ntt3.cu k_ks3): one
        task per (ciphertext, target row)."""
        if len(tasks):
            d = _upload(tasks, self.device)
            e0 = _STATS.begin() if _STATS else None
            nat.check(self._lib.hb_ks_fused(self.handle, _ptr(d), len(tasks), self.stream),
                      "ks_fused")
            if _STATS:   # digit rows once, identity rows, key rows once, two outputs per task
                _STATS.end("keyswitch_fused", e0)
                m = len(tasks)
                ndig = tasks["ndig"].astype(np.int64)
                lifts = int((ndig - (tasks["ident_digit"] >= 0)).sum())
                keys = len({(int(a), int(n)) for a, n in zip(tasks["kb"], tasks["ndig"])})
                nd = int(ndig.max())
                nbytes = (_uniq(tasks["coef"]) * nd + _uniq(tasks["ident"]) + 2 * keys * nd
                          + 2 * m) * 8 * self.n + lifts * 16 * self.n // 8
                fp64 = lifts * (self.n // 2) * self.logn * StepStats.FP64_PER_BUTTERFLY \
                    + 2 * int(ndig.sum()) * self.n * StepStats.FP64_PER_MODMUL
                _STATS.add("keyswitch_fused", nbytes, fp64)

    def rot_sum(self, tasks: np.ndarray, rots: np.ndarray, ndig: int, nb: int):
        """ct + sum_j rot_j(ct) in the extended basis (csrc/ops.cu k_rot_sum_f64)."""
        if len(tasks):
            d, r = _upload(tasks, self.device), _upload(rots, self.device)
            e0 = _STATS.begin() if _STATS else None
            nat.check(self._lib.hb_rot_sum(self.handle, _ptr(d), len(tasks), _ptr(r), len(rots),
                                           ndig, nb, self.stream), "rot_sum")
            if _STATS:   # digit rows and c rows once, key rows once, two outputs per task
                _STATS.end("rot_sum", e0)
                m = len(tasks)
                nrows = len(set(tasks["prime"].tolist()))
                nbytes = (m * nb * (ndig + 4) + 2 * len(rots) * ndig * nrows) * 8 * self.n
                _STATS.add("rot_sum", nbytes, 2 * m * nb * len(rots) * ndig * self.n
                           * StepStats.FP64_PER_MODMUL)

    def ks_inner2(self, tasks: np.ndarray, nb: int):
        if len(tasks):
            d = _upload(tasks, self.device)
            nat.check(self._lib.hb_ks_inner2(self.handle, _ptr(d), len(tasks), nb, self.stream),
                      "ks_inner2")

    # ---- row-pointer helpers ---------------------------------------------------

    def row_ptrs(self, t: torch.Tensor) -> np.ndarray:
        """Base addresses of every row of a contiguous (..., R, N) tensor, in
        row-major order (flattened leading dims)."""
        assert t.is_contiguous() and t.shape[-1] == self.n
        rows = t.numel() // self.n
        return np.uint64(t.data_ptr()) + np.arange(rows, dtype=np.uint64) * np.uint64(8 * self.n)

    def zeros(self, *shape) -> torch.Tensor:
        return torch.zeros(*shape, self.n, dtype=torch.int64, device=self.device)

    def empty(self, *shape) -> torch.Tensor:
        return torch.empty(*shape, self.n, dtype=torch.int64, device=self.device)


def _powers(base: int, exps: np.ndarray, q: int) -> np.ndarray:
    """base^e mod q for every e in exps (exact, via a power table)."""
    n = len(exps)
    pw = np.empty(2 * n, dtype=object)
    acc = 1
    for e in range(2 * n):
        pw[e] = acc
        acc = acc * base % q
    return np.array([pw[int(e)] for e in exps], dtype=np.uint64)


def shoup_np(w: np.ndarray, p: np.ndarray) -> np.ndarray:
    w = np.broadcast_to(np.asarray(w, dtype=object), np.broadcast(w, p).shape)
    p = np.broadcast_to(np.asarray(p, dtype=object), w.shape)
    return np.array([(int(a) << 64) // int(b) for a, b in zip(w.ravel(), p.ravel())],
                    dtype=np.uint64).reshape(w.shape)
