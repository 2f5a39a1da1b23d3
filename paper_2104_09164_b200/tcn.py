"""Temporal-convolution HEAR variants: BASELINE configs 0 and 3.

The reference's `NetworkShape` fixes three same-padded kernel-3 conv blocks,
window-2 pooling and degree-2 collapsed activations
(hear/model.py:24-42, convolution.py:108-120).  BASELINE names two networks
outside that family:

  config 0  conv1d over the 30 joint-coordinate channels (k=8, 32 filters,
            stride 2) -> square -> average pool -> FC to 5 classes,
            weights N(0, 0.1);
  config 3  conv1d (k=8, 64 filters) -> square -> conv1d (k=4, 64 filters)
            -> degree-3 polynomial activation -> average pool -> FC to 10
            classes, weights N(0, 0.05), at N = 2^16.

This module is the API extension that expresses them: `TcnShape` (any
stack of valid-padded temporal convolutions with kernel, filters and stride
per layer, a square or cubic activation after each, global average pooling
and a fully connected readout), its cleartext oracle `infer_clear_tcn`, and
an encrypted schedule `compile_tcn` / `TcnEncoder` / `run_tcn` written
against the same backend contract as the reference pipeline
(hear/backend.py), so it runs unchanged on the slot simulator and on the
GPU engine, with per-layer counters.

Packing: channel c of a layer lives in slot block c (B = pot(frames)
slots), time step t at offset t * ts inside the block (ts = product of the
strides so far); one ciphertext holds n2 / B blocks, so every layer of both
networks is ONE ciphertext handle (which may carry a batch of clips).

Convolution (valid padding, stride s), baby-step / giant-step over the
slot-block offset d = c_in - f_out = g D + e (0 <= e < g; the rotate-and-
sum of HEAR §3.2 with the giant/baby refinement of §3.4, Eqs. 3-4):

    y = sum_D rot( sum_{e,k} W''_{D,e,k} * rot(x, e B + k ts), g D B )

with W''_{D,e,k}[(f + g D) B + s t' ts] = W[f, f + g D + e, k] for every
valid output t': K g - 1 hoisted baby rotations of the input (one ModUp),
one giant rotation per D, one plaintext product per nonzero (D, e, k).  The
baby width g minimises (K g) x (hoisted cost) + (#D) x (full key-switch
cost): a hoisted rotation costs the ModDown (2 (l+1) NTTs), a giant one
ModUp + ModDown ((l+1)(l+2) + 2 (l+1) NTTs).  Weights are zero off the output lattice
and outside the filter range, so every slot outside the valid lattice stays
EXACTLY zero through the network (no masks), which lets the polynomial
activation add its constant term only on the lattice and lets the pooling
sum whole blocks.  Every plaintext is encoded at the scale that returns
the product to the network scale Delta after the rescale (level-aware
encoding, HEAR §4.2), so conv / mask / FC outputs sit at exactly Delta.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from .backend import BackendBase, Ct
from .layout import pot


@dataclass(frozen=True)
class ConvSpec:
    kernel: int
    filters: int
    stride: int = 1


@dataclass(frozen=True)
class TcnShape:
    """A stack of valid temporal convolutions over the 2*joints coordinate
    channels of a (frames, joints, 2) clip, activation `acts[i]` after conv
    i ("square": x^2, "poly3": a0 + a1 x + a2 x^2 + a3 x^3), global average
    pooling over time, FC to `classes`."""

    frames: int
    joints: int
    convs: tuple
    acts: tuple
    classes: int

    def __post_init__(self):
        if len(self.convs) != len(self.acts) or not self.convs:
            raise ValueError("one activation per conv layer")
        for a in self.acts:
            if a not in ("square", "poly3"):
                raise ValueError(f"unknown activation '{a}'")
        t = self.frames
        for cv in self.convs:
            if cv.kernel < 1 or cv.stride < 1 or cv.filters < 1:
                raise ValueError("kernel, stride and filters must be positive")
            t = (t - cv.kernel) // cv.stride + 1
            if t < 1:
                raise ValueError("sequence shorter than the kernel")
        if pot(self.classes) > self.block:
            raise ValueError("more classes than slots per block")

    @property
    def channels_in(self) -> int:
        return 2 * self.joints

    @property
    def block(self) -> int:
        return pot(self.frames)

    def lengths(self) -> list:
        """Sequence length after each conv (input first)."""
        out = [self.frames]
        for cv in self.convs:
            out.append((out[-1] - cv.kernel) // cv.stride + 1)
        return out

    def channels(self) -> list:
        return [self.channels_in] + [cv.filters for cv in self.convs]


TCN_NETS = {
    "config0": TcnShape(32, 15, (ConvSpec(8, 32, 2),), ("square",), 5),
    "config3": TcnShape(32, 15, (ConvSpec(8, 64, 1), ConvSpec(4, 64, 1)), ("square", "poly3"), 10),
}
TCN_WEIGHT_STD = {"config0": 0.1, "config3": 0.05}

GIANT_GROUP = 16

# cubic activation of config 3 (BASELINE names only its degree): a fixed
# smooth, non-odd polynomial, so the constant and every power are exercised
POLY3 = (0.05, 0.5, 0.25, 0.1)


def tcn_by_name(name: str) -> TcnShape:
    if name not in TCN_NETS:
        raise KeyError(f"unknown temporal network '{name}' (have {sorted(TCN_NETS)})")
    return TCN_NETS[name]


@dataclass
class TcnParams:
    shape: TcnShape
    filters: list            # per conv: (filters, channels_in, kernel)
    act: list                # per conv: None (square) or (a0, a1, a2, a3)
    fc_w: np.ndarray         # (classes, filters of the last conv)
    fc_b: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def validate(self):
        s = self.shape
        for i, cv in enumerate(s.convs):
            want = (cv.filters, s.channels()[i], cv.kernel)
            if self.filters[i].shape != want:
                raise ValueError(f"conv{i + 1} filters must be {want}")
        if self.fc_w.shape != (s.classes, s.convs[-1].filters):
            raise ValueError("fc matrix shape mismatch")
        if self.fc_b.size == 0:
            self.fc_b = np.zeros(s.classes)


def make_random_tcn(shape: TcnShape, seed: int, std: float) -> TcnParams:
    """Weights N(0, std) from `seed` (BASELINE configs 0 / 3)."""
    rng = np.random.default_rng(seed)
    filt = [rng.normal(0.0, std, (cv.filters, ch, cv.kernel))
            for cv, ch in zip(shape.convs, shape.channels())]
    fc = rng.normal(0.0, std, (shape.classes, shape.convs[-1].filters))
    act = [None if a == "square" else POLY3 for a in shape.acts]
    p = TcnParams(shape, filt, act, fc)
    p.validate()
    return p


def make_random_clip(shape: TcnShape, seed: int) -> np.ndarray:
    """(frames, joints, 2) uniform[-1, 1] from `seed` (BASELINE config 0 input)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, (shape.frames, shape.joints, 2))


def _channels_time(x: np.ndarray) -> np.ndarray:
    """(T, J, 2) -> (2J, T): channel c = 2 j + coordinate."""
    t = x.shape[-3]
    return np.swapaxes(x.reshape(*x.shape[:-3], t, -1), -1, -2)


def infer_clear_tcn(p: TcnParams, x: np.ndarray) -> np.ndarray:
    """Cleartext oracle: valid conv1d stack, activations, global average
    pooling over time, FC (+ bias).  x: (T, J, 2)."""
    h = _channels_time(np.asarray(x, dtype=np.float64))
    for cv, w, act in zip(p.shape.convs, p.filters, p.act):
        tout = (h.shape[1] - cv.kernel) // cv.stride + 1
        y = np.zeros((cv.filters, tout))
        for k in range(cv.kernel):
            y += w[:, :, k] @ h[:, k:k + cv.stride * (tout - 1) + 1:cv.stride]
        h = y * y if act is None else act[0] + y * (act[1] + y * (act[2] + y * act[3]))
    return p.fc_w @ h.mean(axis=1) + p.fc_b


# ---- encrypted schedule ----------------------------------------------------------

@dataclass
class TcnStep:
    name: str
    level: int
    scale: Fraction


@dataclass
class TcnPlan:
    """Static schedule of a TcnShape at a parameter set: per conv the slot
    stride, lengths and the giant-step offsets; the level / scale of every
    step; the rotation keys {amount: max level}."""
    shape: TcnShape
    params: object
    delta: Fraction
    ts: list                          # slot stride of the time axis per layer (input first)
    offsets: list                     # per conv: block offsets d = c_in - f_out
    bsgs: list = field(default_factory=list)   # per conv: (g, [giant D], {D: [(e, k)]})
    steps: dict = field(default_factory=dict)
    rotations: dict = field(default_factory=dict)

    def expected(self, name: str) -> TcnStep:
        return self.steps[name]

    @property
    def levels_used(self) -> int:
        return self.params.max_level - self.steps["fc"].level


def _need_rot(rot: dict, amount: int, level: int, n2: int):
    a = amount % n2
    if a:
        rot[a] = max(rot.get(a, -1), level)


def _bsgs_split(offs, kernel: int, lvl: int):
    """(g, giant steps D, {D: [(e, k)]}) covering every block offset
    d = g D + e of `offs` with the fewest NTT-equivalents: baby rotations
    are hoisted (ModDown: 2 (l+1) NTTs each), giant ones full key switches
    ((l+1)(l+2) ModUp + 2 (l+1) ModDown NTTs)."""
    r = lvl + 1
    best = None
    for g in range(1, 33):
        ds = sorted({d // g for d in offs})   # floor division: e = d - g D in [0, g)
        cost = (kernel * g) * 2 * r + len([D for D in ds if D]) * (r * (r + 1) + 2 * r)
        if best is None or cost < best[0]:
            best = (cost, g, ds)
    _, g, ds = best
    terms = {D: sorted({(d - g * D, k) for d in offs if d // g == D for k in range(kernel)})
             for D in ds}
    return g, ds, terms


def compile_tcn(shape: TcnShape, params) -> TcnPlan:
    """Levels, scales and rotation amounts of the encrypted TCN at `params`."""
    n2, B = params.n2, shape.block
    if shape.frames > B or max(shape.channels()) * B > n2:
        raise ValueError("network does not fit one ciphertext per layer at this ring")
    delta = Fraction(params.msg_scale)
    lens, chans = shape.lengths(), shape.channels()
    ts = [1]
    for cv in shape.convs:
        ts.append(ts[-1] * cv.stride)
    if pot(lens[-1]) * ts[-1] > B:
        raise ValueError("pooled lattice exceeds the slot block")
    plan = TcnPlan(shape, params, delta, ts, [])
    rot: dict = {}
    lvl = params.max_level
    plan.steps["input"] = TcnStep("input", lvl, delta)
    prime = params.chain_primes
    scale = delta
    for i, cv in enumerate(shape.convs):
        cin = chans[i]
        offs = sorted({c - f for c in range(cin) for f in range(cv.filters)})
        plan.offsets.append(offs)
        g, giants, terms = _bsgs_split(offs, cv.kernel, lvl)
        plan.bsgs.append((g, giants, terms))
        for e in range(g):
            for k in range(cv.kernel):
                _need_rot(rot, e * B + k * ts[i], lvl, n2)
        for D in giants:
            _need_rot(rot, g * D * B, lvl, n2)
        lvl -= 1                                   # conv rescale -> scale delta
        scale = delta
        plan.steps[f"conv{i + 1}"] = TcnStep(f"conv{i + 1}", lvl, scale)
        if shape.acts[i] == "square":
            scale = scale * scale / prime[lvl]
            lvl -= 1
        else:                                      # poly3: x^2, x^3, coefficients
            lvl -= 3
            scale = delta
        plan.steps[f"act{i + 1}"] = TcnStep(f"act{i + 1}", lvl, scale)
    # global pool: rotate-and-sum over pot(T_last) lattice points
    for b in range((pot(lens[-1]) - 1).bit_length()):
        _need_rot(rot, (1 << b) * ts[-1], lvl, n2)
    plan.steps["pool"] = TcnStep("pool", lvl, scale)
    lvl -= 1                                       # block mask -> delta
    for b in range((pot(shape.classes) - 1).bit_length()):
        _need_rot(rot, -(1 << b), lvl, n2)         # spread over the class slots
    lvl -= 1                                       # FC weights -> delta
    for b in range((pot(shape.convs[-1].filters) - 1).bit_length()):
        _need_rot(rot, (1 << b) * B, lvl, n2)      # sum over filter blocks
    if lvl < 0:
        raise ValueError(f"network needs {params.max_level - lvl} levels, chain has "
                         f"{params.max_level}")
    plan.steps["fc"] = TcnStep("fc", lvl, delta)
    plan.rotations = rot
    return plan


class TcnEncoder:
    """Plaintexts of a TcnParams bound to a TcnPlan, encoded level-aware
    (each at the level it is consumed and at the scale that returns the
    product to Delta after the rescale)."""

    def __init__(self, plan: TcnPlan, tparams: TcnParams, backend: BackendBase):
        if tparams.shape != plan.shape:
            raise ValueError("parameters do not match the plan")
        tparams.validate()
        self.compiled = plan
        self.model = tparams
        self.backend = backend
        self._pts: dict = {}

    def _enc(self, vectors, level: int, scale) -> list:
        vectors = np.asarray(vectors, dtype=np.float64)
        enc = getattr(self.backend, "encode_many", None)
        if enc is not None:
            return enc(vectors, level, scale)
        return [self.backend.encode(v, level, scale) for v in vectors]

    def _pscale(self, level: int, in_scale: Fraction) -> Fraction:
        """Plaintext scale s.t. rescale(ct(in_scale) * pt) has scale Delta."""
        return self.compiled.delta * self.compiled.params.chain_primes[level] / in_scale

    def _in_scale(self, i: int) -> Fraction:
        return self.compiled.expected("input" if i == 0 else f"act{i}").scale

    def _in_level(self, i: int) -> int:
        return self.compiled.expected("input" if i == 0 else f"act{i}").level

    def conv_pts(self, i: int) -> dict:
        """{(D, e, k): plaintext W''} of conv i (0-based): value
        W[f, f + g D + e, k] at block f + g D on the output lattice."""
        key = ("conv", i)
        if key not in self._pts:
            pl, sh = self.compiled, self.compiled.shape
            cv, w = sh.convs[i], self.model.filters[i]
            n2, B, ts = pl.params.n2, sh.block, pl.ts[i]
            tout = sh.lengths()[i + 1]
            cin = sh.channels()[i]
            lattice = np.arange(tout) * cv.stride * ts
            g, giants, terms = pl.bsgs[i]
            keys, vecs = [], []
            for D in giants:
                for e, k in terms[D]:
                    d = g * D + e
                    fs = np.arange(max(-d, 0), min(cv.filters, cin - d))   # c = f + d valid
                    v = np.zeros(n2)
                    for f in fs:
                        v[(f + g * D) % (n2 // B) * B + lattice] = w[f, f + d, k]
                    keys.append((D, e, k))
                    vecs.append(v)
            lvl = self._in_level(i)
            pts = self._enc(vecs, lvl, self._pscale(lvl, self._in_scale(i)))
            self._pts[key] = dict(zip(keys, pts))
        return self._pts[key]

    def act_pts(self, i: int):
        """poly3 of conv i: ([a1, a2, a3] coefficient plaintexts at the level
        of the final products, constant term a0 on the valid lattice)."""
        key = ("act", i)
        if key not in self._pts:
            pl, sh = self.compiled, self.compiled.shape
            a0, a1, a2, a3 = self.model.act[i]
            n2, B = pl.params.n2, sh.block
            x = pl.expected(f"conv{i + 1}")
            l0, s1 = x.level, x.scale
            p = pl.params.chain_primes
            s2 = s1 * s1 / p[l0]                         # x^2 at l0 - 1
            s3 = s2 * s1 / p[l0 - 1]                     # x^3 at l0 - 2
            lf = l0 - 2
            coef = [self._enc([np.full(n2, a)], lf, self._pscale(lf, s))[0]
                    for a, s in ((a1, s1), (a2, s2), (a3, s3))]
            lattice = np.zeros(n2)
            tout, ts = sh.lengths()[i + 1], pl.ts[i + 1]
            for f in range(sh.convs[i].filters):
                lattice[f * B + np.arange(tout) * ts] = a0
            const = self._enc([lattice], lf - 1, pl.delta)[0]
            self._pts[key] = (coef, const)
        return self._pts[key]

    def fc_pts(self):
        """(block mask, FC weights): mask keeps slot f*B of every filter block;
        weights put fc_w[j, f] / T_last at slot f*B + j (average divisor
        folded in)."""
        if "fc" not in self._pts:
            pl, sh = self.compiled, self.compiled.shape
            n2, B = pl.params.n2, sh.block
            F = sh.convs[-1].filters
            st = pl.expected("pool")
            mask = np.zeros(n2)
            mask[np.arange(F) * B] = 1.0
            m = self._enc([mask], st.level, self._pscale(st.level, st.scale))[0]
            w = np.zeros(n2)
            tl = sh.lengths()[-1]
            for j in range(sh.classes):
                w[np.arange(F) * B + j] = self.model.fc_w[j] / tl
            wl = st.level - 1
            wp = self._enc([w], wl, self._pscale(wl, pl.delta))[0]
            self._pts["fc"] = (m, wp)
        return self._pts["fc"]

    def prepare(self):
        """Encode every plaintext now (setup, not per clip)."""
        for i, a in enumerate(self.compiled.shape.acts):
            self.conv_pts(i)
            if a == "poly3":
                self.act_pts(i)
        self.fc_pts()
        return self


def _check(ct: Ct, plan: TcnPlan, name: str):
    st = plan.expected(name)
    if ct.level != st.level or ct.scale != st.scale:
        raise ValueError(f"{name}: at (level {ct.level}, scale {float(ct.scale):.6g}), "
                         f"plan says ({st.level}, {float(st.scale):.6g})")


def _rot_sum(ct: Ct, step: int, count: int, backend: BackendBase) -> Ct:
    for b in range((count - 1).bit_length()):
        ct = backend.rot_add_each([(ct, (1 << b) * step)])[0]
    return ct


def run_tcn(encoder: TcnEncoder, ct: Ct, backend: BackendBase) -> Ct:
    """Evaluate the encrypted TCN on one input handle (any batch of clips);
    returns the logits handle (logit j at slot j)."""
    pl, sh = encoder.compiled, encoder.compiled.shape
    B = sh.block
    _check(ct, pl, "input")
    for i, cv in enumerate(sh.convs):
        with backend.layer(f"conv{i + 1}"):
            ts = pl.ts[i]
            pts = encoder.conv_pts(i)
            g, giants, terms = pl.bsgs[i]
            # the baby steps only feed the inner sums: their ModDown may be
            # deferred to one per inner sum
            baby = backend.rot_many_each([ct], [e * B + k * ts for e in range(g)
                                                for k in range(cv.kernel)], lazy=True)[0]
            acc = None
            # giant steps in groups of GIANT_GROUP: the inner sums of one
            # group are live at a time (B clips x rows per handle); same op
            # counts as one flat sum
            for g0 in range(0, len(giants), GIANT_GROUP):
                grp = giants[g0:g0 + GIANT_GROUP]
                inner = backend.mac_many([[(baby[(e * B + k * ts) % backend.n2], pts[(D, e, k)])
                                           for e, k in terms[D]] for D in grp])
                giant = backend.rot_each([(x, g * D * B) for x, D in zip(inner, grp)], lazy=True)
                part = backend.sum_each([giant])[0]
                acc = part if acc is None else backend.add(acc, part)
            ct = backend.rescale(acc)
        _check(ct, pl, f"conv{i + 1}")
        with backend.layer(f"act{i + 1}"):
            if sh.acts[i] == "square":
                ct = backend.square_rescale_each([ct])[0]
            else:
                (c1, c2, c3), const = encoder.act_pts(i)
                x2 = backend.square_rescale_each([ct])[0]
                x3 = backend.rescale(backend.mult(x2, backend.mod_down(ct, x2.level)))
                lf = x3.level
                # x, x^2, x^3 carry different scales, so each coefficient is
                # its own plaintext product; they meet at Delta after rescale
                prods = backend.mac_many([[(backend.mod_down(ct, lf), c1)],
                                          [(backend.mod_down(x2, lf), c2)], [(x3, c3)]])
                prods = backend.rescale_each(prods)
                ct = backend.add_plain(backend.sum_each([prods])[0], const)
        _check(ct, pl, f"act{i + 1}")
    with backend.layer("pool"):
        ct = _rot_sum(ct, pl.ts[-1], pot(sh.lengths()[-1]), backend)
    _check(ct, pl, "pool")
    with backend.layer("fc"):
        mask, w = encoder.fc_pts()
        ct = backend.rescale(backend.mult_plain(ct, mask))
        ct = _rot_sum(ct, -1, pot(sh.classes), backend)
        ct = backend.rescale(backend.mult_plain(ct, w))
        ct = _rot_sum(ct, B, pot(sh.convs[-1].filters), backend)
    _check(ct, pl, "fc")
    return ct


def pack_tcn_input(x: np.ndarray, plan: TcnPlan) -> np.ndarray:
    """(T, J, 2) or (B, T, J, 2) -> slot vectors: channel c, time t at c*B + t."""
    x = np.asarray(x, dtype=np.float64)
    ct = _channels_time(x)                             # (..., C, T)
    n2, B = plan.params.n2, plan.shape.block
    out = np.zeros(ct.shape[:-2] + (n2,))
    C, T = ct.shape[-2:]
    if (C, T) != (plan.shape.channels_in, plan.shape.frames):
        raise ValueError("input tensor does not match the network")
    idx = (np.arange(C)[:, None] * B + np.arange(T)[None, :]).ravel()
    out[..., idx] = ct.reshape(*ct.shape[:-2], -1)
    return out


def encrypt_tcn_input(x: np.ndarray, plan: TcnPlan, backend: BackendBase) -> Ct:
    return backend.enc(pack_tcn_input(x, plan), level=plan.params.max_level, scale=plan.delta)


def dec_tcn_logits(out: Ct, encoder: TcnEncoder, backend: BackendBase) -> np.ndarray:
    vals = backend.dec(out)
    return vals[..., :encoder.compiled.shape.classes] + encoder.model.fc_b


def infer_tcn(tparams: TcnParams, x: np.ndarray, backend: BackendBase, encoder=None):
    """(logits, counters, encoder) of one clip or a batch of clips."""
    if encoder is None:
        encoder = TcnEncoder(compile_tcn(tparams.shape, backend.params), tparams, backend)
    out = run_tcn(encoder, encrypt_tcn_input(x, encoder.compiled, backend), backend)
    return dec_tcn_logits(out, encoder, backend), backend.counters, encoder
