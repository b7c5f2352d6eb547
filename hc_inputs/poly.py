"""Tiny sparse polynomial algebra over C in unknowns x (n) and parameters p (P).

Used only to *write down* the polynomial systems of PAPER.md §4 and Table 1 and
expand them into term lists; it is problem-formulation plumbing, not part of the
HC method.  A polynomial is a dict {(x-exponents..., p-exponents...): complex}.
"""
from __future__ import annotations


class Poly:
    __slots__ = ("n", "P", "t")

    def __init__(self, n: int, P: int, terms=None):
        self.n, self.P = n, P
        self.t = {} if terms is None else terms

    # -- construction -------------------------------------------------
    def copy(self):
        return Poly(self.n, self.P, dict(self.t))

    def _coerce(self, o):
        if isinstance(o, Poly):
            assert (o.n, o.P) == (self.n, self.P)
            return o
        return const(self.n, self.P, o)

    # -- ring operations ----------------------------------------------
    def __add__(self, o):
        o = self._coerce(o)
        r = dict(self.t)
        for k, v in o.t.items():
            w = r.get(k, 0) + v
            if w == 0:
                r.pop(k, None)
            else:
                r[k] = w
        return Poly(self.n, self.P, r)

    __radd__ = __add__

    def __neg__(self):
        return Poly(self.n, self.P, {k: -v for k, v in self.t.items()})

    def __sub__(self, o):
        return self + (-self._coerce(o))

    def __rsub__(self, o):
        return self._coerce(o) - self

    def __mul__(self, o):
        o = self._coerce(o)
        r = {}
        for k1, v1 in self.t.items():
            for k2, v2 in o.t.items():
                k = tuple(a + b for a, b in zip(k1, k2))
                w = r.get(k, 0) + v1 * v2
                if w == 0:
                    r.pop(k, None)
                else:
                    r[k] = w
        return Poly(self.n, self.P, r)

    __rmul__ = __mul__

    def __pow__(self, e: int):
        r = const(self.n, self.P, 1)
        for _ in range(e):
            r = r * self
        return r

    def diff_x(self, i: int):
        """Partial derivative with respect to unknown x_i (exponent decrement)."""
        r = {}
        for k, v in self.t.items():
            e = k[i]
            if e:
                kk = list(k)
                kk[i] -= 1
                kk = tuple(kk)
                r[kk] = r.get(kk, 0) + v * e
        return Poly(self.n, self.P, {k: v for k, v in r.items() if v != 0})

    def degree_x(self):
        return max((sum(k[: self.n]) for k in self.t), default=0)

    def __repr__(self):
        return f"Poly(n={self.n}, P={self.P}, terms={len(self.t)})"


def const(n: int, P: int, c) -> Poly:
    c = complex(c)
    return Poly(n, P, {} if c == 0 else {(0,) * (n + P): c})


def var_x(n: int, P: int, i: int) -> Poly:
    k = [0] * (n + P)
    k[i] = 1
    return Poly(n, P, {tuple(k): 1 + 0j})


def var_p(n: int, P: int, q: int) -> Poly:
    k = [0] * (n + P)
    k[n + q] = 1
    return Poly(n, P, {tuple(k): 1 + 0j})
