"""Homomorphic convolution over packed slots (restates hear/convolution.py).

A conv layer consumes n_I ciphertexts of ell channel blocks and emits n_O
ciphertexts whose block b holds output channel j*ell_O + b.  Each output sums
MultPlain(rot(ct_i, r_k + block*l), pt[i,j,k,l]) over inputs i, taps k and
block alignments l; the strategies only choose which handle is rotated:

  full   pre-rotate every r_k + block*l per input   (one hoisted group / input)
  giant  pre-rotate block*l; rotate partial sums by r_k   (counter-rotated pts)
  baby   pre-rotate r_k; rotate partial sums by block*l   (counter-rotated pts)

The B200 schedule issues the same contract ops layer-wide: every partial sum
of the layer is one multiply-accumulate launch (BackendBase.mac_many), every
partial-sum rotation one batched key switch (rot_each), then one batched add
and one batched rescale -- identical values and counters to the reference's
op-by-op path (hear/convolution.py:247-312), since modular sums are exact.
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from .backend import BackendBase, Ct
from .layout import PackedLayout


@dataclass(frozen=True)
class MergeGrid:
    n_p: int
    n_cols: int
    n_rows: int


@dataclass
class ConvPlan:
    t: int
    strategy: str
    layout_in: PackedLayout
    merge: MergeGrid | None
    taps: list
    n_i: int
    n_o: int
    ell_i: int
    ell_o: int
    c_in: int
    c_out: int

    @property
    def n_p(self) -> int:
        return self.merge.n_p if self.merge else 1

    @property
    def m(self) -> int:
        return self.n_i // self.n_p

    @property
    def block(self) -> int:
        return self.layout_in.block

    @property
    def tap_amounts(self) -> list:
        lay = self.layout_in
        return [(dy * lay.map_w + dx) * lay.stride for dy, dx in self.taps]

    @property
    def f(self) -> int:
        return len(self.taps)

    @property
    def block_amounts(self) -> list:
        return [self.block * l for l in range(self.ell_i)]

    def rotation_amounts(self) -> set:
        taps, blocks = self.tap_amounts, self.block_amounts
        if self.strategy == "full":
            amts = {r + b for r in taps for b in blocks}
        elif self.strategy in ("giant", "baby"):
            amts = set(taps) | set(blocks)
        else:
            raise ValueError(f"unknown strategy '{self.strategy}'")
        n2 = self.layout_in.n2
        return {a % n2 for a in amts if a % n2}

    def pre_amounts(self) -> list:
        """Hoisted rotations applied to every input ciphertext."""
        taps, blocks = self.tap_amounts, self.block_amounts
        if self.strategy == "full":
            return [r + b for r in taps for b in blocks]
        return blocks if self.strategy == "giant" else taps

    def describe(self) -> dict:
        return {"layer": f"conv{self.t}", "strategy": self.strategy, "n_I": self.n_i,
                "n_O": self.n_o, "n_P": self.n_p, "ell_I": self.ell_i, "ell_O": self.ell_o,
                "taps": self.tap_amounts, "rotations": sorted(self.rotation_amounts())}


def make_plan(t: int, shape, layout_in: PackedLayout, strategy: str,
              merge: MergeGrid | None = None) -> ConvPlan:
    ell = layout_in.channels_per_ct
    c_in, c_out = shape.channels_in(t), shape.channels_out(t)
    n_i, ell_i = (1, c_in) if t == 1 else (-(-c_in // ell), ell)
    return ConvPlan(t=t, strategy=strategy, layout_in=layout_in, merge=merge, taps=shape.taps,
                    n_i=n_i, n_o=-(-c_out // ell), ell_i=ell_i, ell_o=ell, c_in=c_in,
                    c_out=c_out)


class _Geometry:
    """Block-periodic slot masks of one conv input layout."""

    def __init__(self, plan: ConvPlan):
        lay = plan.layout_in
        q = np.arange(lay.block)
        row, col = q // lay.map_w, q % lay.map_w
        pad = q >= lay.map_h * lay.map_w
        s = lay.stride
        dr, dc = row % s, col % s
        self.n_rows, self.n_cols = (plan.merge.n_rows, plan.merge.n_cols) if plan.merge else (1, 1)
        ok = ~pad & (dr < self.n_rows) & (dc < self.n_cols)
        br, bc = (row - dr) // s, (col - dc) // s
        self.src = np.where(ok, dr * self.n_cols + dc, -1)
        self.out_valid = ok & (br < lay.cur_h) & (bc < lay.cur_w)
        self.tap_ok = np.stack([
            self.out_valid & (br + dy >= 0) & (br + dy < lay.cur_h)
            & (bc + dx >= 0) & (bc + dx < lay.cur_w) for dy, dx in plan.taps])


class ConvWeights:
    """Weight plaintexts of one conv layer.

    Slot s of pt[i, j, k, l] holds F[out(s), in(s, i, l), k] when s is a
    partial-result position of its source lattice and tap k lands in-map,
    else 0 (hear/convolution.py:152-229); giant/baby tables are the
    counter-rotated full tables.  Tables are encoded per output block,
    all f*ell_i*m plaintexts of a block in one batched encode."""

    def __init__(self, filters, plan: ConvPlan, backend: BackendBase, level: int,
                 scale: Fraction, cache: bool = True):
        self.filters = np.asarray(filters, dtype=np.float64)
        self.plan = plan
        self.backend = backend
        self.level = level
        self.scale = scale
        self.cache = cache
        self._cached: dict = {}
        self.geom = _Geometry(plan)

    def pt_count(self) -> int:
        p = self.plan
        return p.f * p.ell_i * p.m * p.n_o

    def values(self, j: int) -> np.ndarray:
        """All slot vectors of output block j as (m, ell_i, f, n2), already
        counter-rotated for the giant / baby strategies."""
        p, g = self.plan, self.geom
        lay = p.layout_in
        per, n2 = lay.channels_per_ct, lay.n2
        blk = np.repeat(np.arange(per), lay.block)
        src = np.tile(g.src, per)
        oc = j * p.ell_o + blk
        out = np.zeros((p.m, p.ell_i, p.f, n2))
        tap_ok = np.tile(g.tap_ok, (1, per))                       # (f, n2)
        ky_of = [0 if self.filters.shape[2] == 1 else dy + 1 for dy, _ in p.taps]
        kx_of = [dx + 1 for _, dx in p.taps]
        for i in range(p.m):
            for l in range(p.ell_i):
                in_blk = (blk + l) % per
                if lay.replicas > 1:
                    ch = in_blk % lay.channels
                else:
                    ch = (i * p.n_p + np.maximum(src, 0)) * per + in_blk
                base = (oc < p.c_out) & (ch < p.c_in) & (src >= 0)
                w = self.filters[np.minimum(oc, p.c_out - 1), np.minimum(ch, p.c_in - 1)]
                for k in range(p.f):
                    v = np.where(base & tap_ok[k], w[:, ky_of[k], kx_of[k]], 0.0)
                    if p.strategy == "giant":
                        v = np.roll(v, p.tap_amounts[k])
                    elif p.strategy == "baby":
                        v = np.roll(v, p.block * l)
                    out[i, l, k] = v
        return out

    def for_output(self, j: int) -> dict:
        """{(i, k, l): Pt} for output block j."""
        if j in self._cached:
            return self._cached[j]
        p = self.plan
        vals = self.values(j)
        flat = vals.reshape(-1, vals.shape[-1])
        enc = getattr(self.backend, "encode_many", None)
        pts = enc(flat, self.level, self.scale) if enc else \
            [self.backend.encode(v, self.level, self.scale) for v in flat]
        table = {}
        q = 0
        for i in range(p.m):
            for l in range(p.ell_i):
                for k in range(p.f):
                    table[(i, k, l)] = pts[q]
                    q += 1
        if self.cache:
            self._cached[j] = table
        return table


def simple_conv(ct: Ct, pts: list, amounts: list, backend: BackendBase) -> Ct:
    """sum_k MultPlain(rot(ct, r_k), pt_k); caller rescales."""
    if len(pts) != len(amounts):
        raise ValueError("one plaintext per tap")
    rots = backend.rot_many(ct, amounts)
    return backend.mac_many([[(rots[r % backend.n2], pt) for r, pt in zip(amounts, pts)]])[0]


def hconv(cts: list, weights: ConvWeights, plan: ConvPlan, backend: BackendBase,
          j_chunk: int | None = None) -> list:
    """Multi-channel convolution of every output block, one rescale each."""
    if len(cts) != plan.m:
        raise ValueError(f"expected {plan.m} input ciphertexts, got {len(cts)}")
    n2 = backend.n2
    taps, blocks = plan.tap_amounts, plan.block_amounts
    # "full": the rotated inputs only feed the accumulations below, so the
    # engine may defer their ModDown past the plaintext products
    pre = backend.rot_many_each(cts, plan.pre_amounts(), lazy=plan.strategy == "full")
    if j_chunk is None:
        j_chunk = plan.n_o
    outs = []
    for j0 in range(0, plan.n_o, j_chunk):
        js = range(j0, min(plan.n_o, j0 + j_chunk))
        jobs, rot_amt, owner = [], [], []
        if plan.strategy == "full":
            # no partial-sum rotations: each output is one accumulation over all
            # f*ell_i*m products (same mult_plain/add counts as the per-tap
            # partials plus their sum, and the same exact modular sum), and
            # every output shares the same hoisted term list -> one MAC group
            fj = []
            for j in js:
                pts = weights.for_output(j)
                fj.append([(pre[i][(taps[k] + blocks[l]) % n2], pts[(i, k, l)])
                           for k in range(plan.f) for l in range(plan.ell_i)
                           for i in range(plan.m)])
            outs += backend.mac_rescale_many(fj)
            continue
        for j in js:
            pts = weights.for_output(j)
            if plan.strategy == "baby":
                for l in range(plan.ell_i):
                    jobs.append([(pre[i][taps[k] % n2], pts[(i, k, l)])
                                 for k in range(plan.f) for i in range(plan.m)])
                    rot_amt.append(blocks[l])
                    owner.append(j)
            else:
                for k in range(plan.f):
                    src = (lambda l: (taps[k] + blocks[l]) % n2) if plan.strategy == "full" \
                        else (lambda l: blocks[l] % n2)
                    jobs.append([(pre[i][src(l)], pts[(i, k, l)])
                                 for l in range(plan.ell_i) for i in range(plan.m)])
                    rot_amt.append(taps[k] if plan.strategy == "giant" else 0)
                    owner.append(j)
        partials = backend.mac_many(jobs)
        moved = backend.rot_each(list(zip(partials, rot_amt)), lazy=True)   # only summed below
        groups = [[c for c, o in zip(moved, owner) if o == j] for j in js]
        outs += backend.rescale_each(backend.sum_each(groups))
    return outs
