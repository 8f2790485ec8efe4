"""Stand-in for the six gmpy2 functions the reference imports.

Used ONLY by tests/golden/make_golden.py, in the build container, to run the
unmodified reference package (gmpy2 is not installed and there is no network).
Every function is exact integer math, so results equal gmpy2's except for the
(vanishing) chance that a probable-prime test disagrees.
"""

import math

mpz = int


def powmod(x, e, m):
    return pow(int(x), int(e), int(m))


def invert(x, m):
    return pow(int(x), -1, int(m))


def gcd(a, b):
    return math.gcd(int(a), int(b))


_SMALL = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53, 59, 61,
          67, 71, 73, 79, 83, 89, 97]


def is_prime(n, reps=25):
    n = int(n)
    if n < 2:
        return False
    for p in _SMALL:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    # deterministic bases for n < 3.3e24, then extra fixed bases
    bases = _SMALL[:13] + [101, 103, 107, 109, 113, 127, 131, 137, 139, 149][:max(0, reps - 13)]
    for a in bases:
        if a % n == 0:
            continue
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


def next_prime(n):
    n = int(n) + 1
    if n <= 2:
        return 2
    if n % 2 == 0:
        n += 1
    while not is_prime(n):
        n += 2
    return n
