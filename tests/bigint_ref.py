"""Independent pure-Python big-integer references used to PIN the oracle.

Nothing here calls oracle/ or the CUDA path; everything is written from the
textbook definitions (schoolbook negacyclic product, direct NTT sum, CRT, floor
division, symbolic substitution, Lucas primality proofs)."""
from __future__ import annotations

import math
import random


def negacyclic_mul(a, b, q):
    """Schoolbook product in Z_q[X]/(X^N+1)."""
    n = len(a)
    c = [0] * n
    for i in range(n):
        ai = int(a[i])
        if ai == 0:
            continue
        for j in range(n):
            k = i + j
            if k < n:
                c[k] += ai * int(b[j])
            else:
                c[k - n] -= ai * int(b[j])
    return [x % q for x in c]


def negacyclic_mul_int(a, b):
    """Schoolbook product over Z[X]/(X^N+1) (no modulus)."""
    n = len(a)
    c = [0] * n
    for i in range(n):
        ai = int(a[i])
        if ai == 0:
            continue
        for j in range(n):
            k = i + j
            if k < n:
                c[k] += ai * int(b[j])
            else:
                c[k - n] -= ai * int(b[j])
    return c


def direct_ntt(a, q, psi):
    """A_k = sum_j a_j psi^{(2k+1) j} mod q, O(N^2)."""
    n = len(a)
    return [sum(int(a[j]) * pow(psi, (2 * k + 1) * j, q) for j in range(n)) % q for k in range(n)]


def substitute(a, kappa):
    """a(X) -> a(X^kappa) mod X^N+1 over Z."""
    n = len(a)
    c = [0] * n
    for j in range(n):
        e = (j * kappa) % (2 * n)
        if e < n:
            c[e] += int(a[j])
        else:
            c[e - n] -= int(a[j])
    return c


def crt(residues, mods):
    Q = math.prod(mods)
    x = 0
    for r, q in zip(residues, mods):
        Qi = Q // q
        x += int(r) * Qi * pow(Qi, -1, q)
    return x % Q


def _trial(n):
    if n < 2:
        return False
    if n % 2 == 0:
        return n == 2
    f = 3
    while f * f <= n:
        if n % f == 0:
            return False
        f += 2
    return True


def _rho(n):
    if n % 2 == 0:
        return 2
    rnd = random.Random(n)
    while True:
        y, c, m = rnd.randrange(1, n), rnd.randrange(1, n), 128
        g = r = q = 1
        while g == 1:
            x = y
            for _ in range(r):
                y = (y * y + c) % n
            k = 0
            while k < r and g == 1:
                ys = y
                for _ in range(min(m, r - k)):
                    y = (y * y + c) % n
                    q = q * abs(x - y) % n
                g = math.gcd(q, n)
                k += m
            r *= 2
        if g == n:
            g = 1
            while g == 1:
                ys = (ys * ys + c) % n
                g = math.gcd(abs(x - ys), n)
        if g != n:
            return g


def factor(n):
    fs = []
    for p in range(2, 1000):
        while n % p == 0:
            fs.append(p)
            n //= p
    stack = [n] if n > 1 else []
    while stack:
        m = stack.pop()
        if prove_prime(m):
            fs.append(m)
        else:
            d = _rho(m)
            stack += [d, m // d]
    return sorted(fs)


def prove_prime(n: int) -> bool:
    """True iff n is prime: trial division below 2^24, else a Lucas certificate
    (a^{n-1} = 1 and a^{(n-1)/p} != 1 for every prime p | n-1), with the factors of
    n-1 proven recursively.  A Fermat witness proves compositeness."""
    if n < (1 << 24):
        return _trial(n)
    ps = sorted(set(factor(n - 1)))
    for a in range(2, 400):
        if pow(a, n - 1, n) != 1:
            return False
        if all(pow(a, (n - 1) // p, n) != 1 for p in ps):
            return True
    raise RuntimeError(f"undecided {n}")
