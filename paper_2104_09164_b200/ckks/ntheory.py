"""Exact integer helpers for parameter generation: deterministic Miller-Rabin,
Pollard-rho factoring, smallest primitive roots, bit reversal."""

from __future__ import annotations

import math
import random

_SMALL = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41)


def is_prime(n: int) -> bool:
    """Deterministic for n < 3.3e24 (bases = first 13 primes)."""
    if n < 2:
        return False
    for p in _SMALL:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in _SMALL:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def _rho(n: int) -> int:
    if n % 2 == 0:
        return 2
    rng = random.Random(n)
    while True:
        c = rng.randrange(1, n)
        f = lambda x: (x * x + c) % n  # noqa: E731
        x = y = rng.randrange(2, n)
        d = 1
        while d == 1:
            x = f(x)
            y = f(f(y))
            d = math.gcd(abs(x - y), n)
        if d != n:
            return d


def prime_factors(n: int) -> set[int]:
    out: set[int] = set()
    for p in (2, 3, 5, 7, 11, 13):
        while n % p == 0:
            out.add(p)
            n //= p
    stack = [n] if n > 1 else []
    while stack:
        m = stack.pop()
        if m == 1:
            continue
        if is_prime(m):
            out.add(m)
            continue
        d = _rho(m)
        stack += [d, m // d]
    return out


def smallest_primitive_root(p: int) -> int:
    """Least generator of (Z/p)^* (the convention sympy.primitive_root uses)."""
    phi = p - 1
    fs = prime_factors(phi)
    g = 2
    while True:
        if all(pow(g, phi // f, p) != 1 for f in fs):
            return g
        g += 1


def root_2n(p: int, two_n: int) -> int:
    """Primitive 2N-th root of unity g^((p-1)/2N) with g the least generator
    (hear/ckks/ring.py:230-232)."""
    if (p - 1) % two_n:
        raise ValueError(f"prime {p} is not 1 mod {two_n}")
    return pow(smallest_primitive_root(p), (p - 1) // two_n, p)


def bit_reverse_table(bits: int):
    import numpy as np
    idx = np.arange(1 << bits, dtype=np.int64)
    out = np.zeros_like(idx)
    for b in range(bits):
        out |= ((idx >> b) & 1) << (bits - 1 - b)
    return out
