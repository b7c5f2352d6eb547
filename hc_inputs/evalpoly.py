"""Direct evaluation of a `Poly` by its defining sum (test helper for pins only).

sum over (x-exps, p-exps) -> w of  w * prod x^e * prod p^e, with Python complex
arithmetic.  Independent of the descriptor expansion and of both evaluators
under test (oracle/ and the CUDA path).
"""
from __future__ import annotations


def eval_poly(f, x, p=()):
    n = f.n
    tot = 0j
    for k, w in f.t.items():
        v = complex(w)
        for i, e in enumerate(k[:n]):
            v *= complex(x[i]) ** e
        for q, e in enumerate(k[n:]):
            v *= complex(p[q]) ** e
        tot += v
    return tot
