"""Seeded model / input generator — a bit-exact port of the reference's
``gen::generate`` and ``gen::random_inputs`` (proj/src/gen.cpp:14-392,
proj/include/polycert/rng.hpp:1-44), so the GPU harness builds the BASELINE
architectures' random-init weights without GMP or the reference.

SplitMix64 (rng.hpp:20-26) is evaluated vectorised: the k-th draw of a
generator seeded with ``s`` is ``mix(s + k * golden)``. Every drawn value is a
dyadic rational and therefore an exact double, equal to what the reference's
``decimal_from_rational`` + ``strtod`` round trip produces.
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np

from .network import Layer, Network

_GOLD = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)
_MASK = (1 << 64) - 1


class Rng:
    """rng.hpp:13-44 (``next``, ``below``, ``irange``), vectorised."""

    def __init__(self, seed: int):
        self.state = int(seed) & _MASK

    def next(self, count: int) -> np.ndarray:
        k = np.arange(1, count + 1, dtype=np.uint64)
        with np.errstate(over="ignore"):
            z = np.uint64(self.state) + k * _GOLD
            z = (z ^ (z >> np.uint64(30))) * _C1
            z = (z ^ (z >> np.uint64(27))) * _C2
            z = z ^ (z >> np.uint64(31))
        self.state = (self.state + count * int(_GOLD)) & _MASK
        return z

    def below(self, n: int, count: int) -> np.ndarray:
        return self.next(count) % np.uint64(n)

    def irange(self, lo: int, hi: int, count: int) -> np.ndarray:
        return lo + self.below(hi - lo + 1, count).astype(np.int64)


def _ceil_log2(n: int) -> int:  # gen.cpp:64-69
    t = 0
    while (1 << t) < n:
        t += 1
    return t


def _draw_weights(rng: Rng, fan_in: int, count: int) -> np.ndarray:
    """draw_weight (gen.cpp:71-78): num in [-64, 64] / (64 * 2^max(0, ceil_log2(fan_in)-1))."""
    num = rng.irange(-64, 64, count)
    shift = max(0, _ceil_log2(max(fan_in, 1)) - 1)
    return num.astype(np.float64) / float(64 << shift)


def _draw_bias(rng: Rng, count: int) -> np.ndarray:
    """draw_bias (gen.cpp:80-84): [-32, 32] / 64."""
    return rng.irange(-32, 32, count).astype(np.float64) / 64.0


class _Builder:  # gen.cpp:88-187
    def __init__(self, seed: int):
        self.rng = Rng(seed)
        self.layers: list[Layer] = []

    def shape(self, i):
        return self.layers[i].out_shape

    def set_input(self, w, h, c):
        if self.layers:
            raise ValueError("arch: duplicate input")
        self.layers.append(Layer(kind="input", preds=[], out_shape=(w, h, c)))

    def add_dense(self, pred, n):
        fan_in = int(np.prod(self.shape(pred)))
        wts = _draw_weights(self.rng, fan_in, n * fan_in).reshape(n, fan_in)
        bias = _draw_bias(self.rng, n)
        self.layers.append(Layer(kind="dense", preds=[pred], weights=wts, bias=bias,
                                 out_shape=(1, 1, n)))
        return len(self.layers) - 1

    def add_conv(self, pred, fw, fh, cout, stride, pad):
        iw, ih, ic = self.shape(pred)
        fan_in = fw * fh * ic
        taps = fw * fh * ic * cout
        filt = _draw_weights(self.rng, fan_in, taps)
        bias = _draw_bias(self.rng, cout)
        nw, nh = iw + 2 * pad - fw, ih + 2 * pad - fh
        if nw < 0 or nh < 0 or nw % stride or nh % stride:
            raise ValueError("arch: conv does not tile its input exactly")
        self.layers.append(Layer(kind="conv", preds=[pred], weights=filt, bias=bias,
                                 fw=fw, fh=fh, sw=stride, sh=stride, pw=pad, ph=pad,
                                 cin=ic, cout=cout,
                                 out_shape=(nw // stride + 1, nh // stride + 1, cout)))
        return len(self.layers) - 1

    def add_relu(self, pred):
        self.layers.append(Layer(kind="relu", preds=[pred], out_shape=self.shape(pred)))
        return len(self.layers) - 1

    def add_join(self, a, b):
        self.layers.append(Layer(kind="residual_join", preds=[a, b], out_shape=self.shape(a)))
        return len(self.layers) - 1


class _Parser:  # gen.cpp:16-60
    def __init__(self, s: str):
        self.s, self.i = s, 0

    def ws(self):
        while self.i < len(self.s) and self.s[self.i].isspace():
            self.i += 1

    def done(self):
        self.ws()
        return self.i >= len(self.s)

    def eat(self, c):
        self.ws()
        if self.i < len(self.s) and self.s[self.i] == c:
            self.i += 1
            return True
        return False

    def expect(self, c):
        if not self.eat(c):
            self.fail(f"expected '{c}'")

    def peek(self):
        self.ws()
        return self.s[self.i] if self.i < len(self.s) else "\0"

    def word(self):
        self.ws()
        b = self.i
        while self.i < len(self.s) and self.s[self.i].isascii() and self.s[self.i].isalpha():
            self.i += 1
        if b == self.i:
            self.fail("expected a keyword")
        return self.s[b:self.i]

    def integer(self):
        self.ws()
        b = self.i
        while self.i < len(self.s) and self.s[self.i].isdigit():
            self.i += 1
        if b == self.i:
            self.fail("expected a number")
        return int(self.s[b:self.i])

    def fail(self, what):
        raise ValueError(f"arch: {what} at offset {self.i}")


def _parse_chain(p: _Parser, b: _Builder, frm: int, top: bool) -> int:  # gen.cpp:189-266
    cur, first = frm, True
    while True:
        if p.done():
            break
        c = p.peek()
        if c in "|)":
            break
        if not first:
            p.expect(";")
        if p.done() or p.peek() in "|)":
            break
        first = False
        if p.peek() == "b" and p.s.startswith("block", p.i):
            p.i += 5
            p.expect("(")
            end_a = _parse_chain(p, b, cur, False)
            p.expect("|")
            end_b = _parse_chain(p, b, cur, False)
            p.expect(")")
            cur = b.add_join(end_a, end_b)
            continue
        kw = p.word()
        if kw == "input":
            if not top or cur >= 0:
                p.fail("'input' must be the first statement")
            w = p.integer(); p.expect("x")
            h = p.integer(); p.expect("x")
            ch = p.integer()
            b.set_input(w, h, ch)
            cur = 0
        elif kw == "conv":
            if cur < 0:
                p.fail("'input' must come first")
            fw = p.integer(); p.expect("x")
            fh = p.integer(); p.expect("x")
            co = p.integer()
            stride, pad = 1, 0
            while p.peek() in ("s", "p"):
                opt = p.word()
                if opt == "s":
                    stride = p.integer()
                elif opt == "p":
                    pad = p.integer()
                else:
                    p.fail(f"unknown conv option '{opt}'")
            cur = b.add_conv(cur, fw, fh, co, stride, pad)
        elif kw == "dense":
            if cur < 0:
                p.fail("'input' must come first")
            cur = b.add_dense(cur, p.integer())
        elif kw == "relu":
            if cur < 0:
                p.fail("'input' must come first")
            cur = b.add_relu(cur)
        elif kw == "skip":
            if top:
                p.fail("'skip' is only valid inside a block branch")
        else:
            p.fail(f"unknown statement '{kw}'")
    return cur


def generate(seed: int, arch: str) -> Network:
    """gen::generate (gen.cpp:268-276)."""
    p = _Parser(arch)
    b = _Builder(seed)
    end = _parse_chain(p, b, -1, True)
    if not p.done():
        p.fail("trailing input")
    if end <= 0:
        raise ValueError("arch: no layers")
    net = Network(b.layers)
    net.validate()
    return net


def random_inputs(seed: int, count: int, dim: int) -> np.ndarray:
    """gen::random_inputs (gen.cpp:278-292): pixels k/256, k ~ U{0..256}."""
    rng = Rng(seed)
    k = rng.below(257, count * dim).astype(np.float64)
    return (k / 256.0).reshape(count, dim)


def decimal_from_fraction(q: Fraction) -> str:
    """decimal_from_rational (proj/src/decimal.cpp:78-119): exact finite expansion."""
    num, den = q.numerator, q.denominator
    rest, twos, fives = den, 0, 0
    while rest % 2 == 0:
        rest //= 2; twos += 1
    while rest % 5 == 0:
        rest //= 5; fives += 1
    if rest != 1:
        raise ValueError("rational has no finite decimal expansion")
    digits = max(twos, fives)
    num *= 2 ** (digits - twos) * 5 ** (digits - fives)
    neg = num < 0
    body = str(abs(num))
    if digits == 0:
        out = body
    else:
        if len(body) <= digits:
            body = "0" * (digits - len(body) + 1) + body
        out = body[:-digits] + "." + body[-digits:]
        out = out.rstrip("0").rstrip(".")
    if neg and out != "0":
        out = "-" + out
    return out


def decimal_from_double(x: float) -> str:
    """Exact decimal string of a (dyadic) double."""
    return decimal_from_fraction(Fraction(float(x)))
