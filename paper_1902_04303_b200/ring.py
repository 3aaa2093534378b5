"""Device-resident ring elements of Z_{2^mod_bits}[x]/(x^N + 1).

Mirrors the reference's ``RingElement`` (hegwas/ring.py:68-209): same constructor,
same canonical representatives in [0, 2^mod_bits), same method names and semantics.
The coefficients live in HBM as a limb-major ``[W][N]`` uint32 array (stored in an
int32 torch tensor, W = ceil(mod_bits/32)); every arithmetic method is one or more
sm_100a kernels behind the C-ABI (include/hegwas_b200.h).  Reading ``coeffs``
downloads to Python ints (test / client use only).

The exact negacyclic product that the reference computes by Kronecker substitution
into one big integer (ring.py:46-58) is computed by the native RNS/NTT engine.  A
ring element may also carry a *compact* view: a two's-complement copy of its centered
representative at a small width (plaintexts, secrets, ephemerals), which lets products
mod 2^k use far fewer NTT primes (mod-2^k products are representative independent,
SURVEY §8a R3).

The host-side samplers and ``derive_rng`` restate ring.py:214-255 draw for draw, so
keys and ciphertexts generated from a ``random.Random`` are identical to the reference's.
"""
from __future__ import annotations

import ctypes
import hashlib
import math
import os
import random

import numpy as np

from . import _lib
from .errors import ParameterError


def _torch():
    import torch

    return torch


def words_for(bits: int) -> int:
    return (bits + 31) >> 5


def ints_to_words(coeffs, bits: int) -> np.ndarray:
    """Python ints (any sign) -> [W][N] uint32, reduced mod 2^bits."""
    w = words_for(bits)
    mask = (1 << bits) - 1
    width = 4 * w
    buf = b"".join((c & mask).to_bytes(width, "little") for c in coeffs)
    arr = np.frombuffer(buf, dtype="<u4").reshape(len(coeffs), w)
    return np.ascontiguousarray(arr.T)


def int64_to_words(vals: np.ndarray, bits: int) -> np.ndarray:
    """Signed int64 values -> [W][N] uint32 two's complement mod 2^bits (vectorised)."""
    vals = np.asarray(vals, dtype=np.int64)
    w = words_for(bits)
    out = np.empty((w, vals.shape[0]), dtype=np.uint32)
    u = vals.view(np.uint64)
    out[0] = (u & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    if w > 1:
        out[1] = (u >> np.uint64(32)).astype(np.uint32)
    if w > 2:
        out[2:] = np.where(vals < 0, np.uint32(0xFFFFFFFF), np.uint32(0))[None, :]
    rem = bits & 31
    if rem:
        out[w - 1] &= np.uint32((1 << rem) - 1)
    return out


def words_to_ints(arr: np.ndarray) -> list[int]:
    """[W][N] uint32 -> list of N nonnegative Python ints."""
    arr = np.asarray(arr, dtype=np.uint32)
    w, n = arr.shape
    raw = np.ascontiguousarray(arr.T).astype("<u4").tobytes()
    width = 4 * w
    return [int.from_bytes(raw[i * width:(i + 1) * width], "little") for i in range(n)]


def _device():
    torch = _torch()
    if not torch.cuda.is_available():
        raise _lib.DeviceError("no CUDA device: the B200 evaluator has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def upload_words(arr: np.ndarray):
    torch = _torch()
    arr = np.ascontiguousarray(arr, dtype=np.uint32)
    if not arr.flags.writeable:
        arr = arr.copy()
    host = torch.from_numpy(arr.view(np.int32))
    if not torch.cuda.is_available():
        return host.to(_device())
    # staged through pinned memory so the copy is stream-ordered instead of synchronising the
    # host with the device (a pageable copy waits for all queued work); the caching host
    # allocator keeps the staging block alive until the copy has run
    return host.pin_memory().to(_device(), non_blocking=True)


def download_words(t) -> np.ndarray:
    return t.detach().cpu().numpy().view(np.uint32)


def reserve_device_bytes(nbytes: int, keep_free: int) -> int:
    """Grow the device ciphertext pool (torch's caching allocator) by ONE segment of up to
    ``nbytes``, leaving at least ``keep_free`` bytes to the library's stream-ordered pool
    (prepared keys, scratch).  The segment goes straight back to the cache, so the thousands
    of ciphertext allocations that follow are carved out of it instead of each calling
    cudaMalloc (0.5-0.75 ms apiece at these sizes, measured in a cold P17 setup).
    Returns the bytes reserved (0 if nothing was needed)."""
    torch = _torch()
    dev = _device()
    free, _ = torch.cuda.mem_get_info(dev)
    cached = torch.cuda.memory_reserved(dev) - torch.cuda.memory_allocated(dev)
    want = min(nbytes - cached, free - keep_free)
    if want < (1 << 30):
        return 0
    want &= ~((2 << 20) - 1)
    try:
        block = torch.empty(want, dtype=torch.uint8, device=dev)
    except torch.OutOfMemoryError:
        return 0
    del block
    return want


def empty_words(bits: int, n: int):
    torch = _torch()
    try:
        return torch.empty((words_for(bits), n), dtype=torch.int32, device=_device())
    except torch.OutOfMemoryError:
        _lib.release_device_memory()   # caches of the library arena / dead keys, then retry
        return torch.empty((words_for(bits), n), dtype=torch.int32, device=_device())


def _ctx(n: int) -> _lib.Context:
    return _lib.get_context(n.bit_length() - 1)


class RingElement:
    """Element of Z_{2^mod_bits}[x]/(x^n + 1), resident in device memory."""

    __slots__ = ("n", "mod_bits", "words", "compact_words", "compact_bits", "__weakref__")

    def __init__(self, n: int, mod_bits: int, coeffs=None, *, _reduced: bool = False,
                 words=None, compact=None):
        if n & (n - 1) or n < 1:
            raise ParameterError(f"ring degree {n} is not a power of two")
        if mod_bits < 1:
            raise ParameterError("modulus must be at least 2^1")
        self.n = n
        self.mod_bits = mod_bits
        self.compact_words = None
        self.compact_bits = 0
        if words is not None:
            if tuple(words.shape) != (words_for(mod_bits), n):
                raise ParameterError(f"word array shape {tuple(words.shape)} != ({words_for(mod_bits)}, {n})")
            self.words = words
        else:
            if coeffs is None or len(coeffs) != n:
                raise ParameterError(f"expected {n} coefficients, got {0 if coeffs is None else len(coeffs)}")
            self.words = upload_words(ints_to_words(coeffs, mod_bits))
        if compact is not None:
            self.compact_words, self.compact_bits = compact

    # -- constructors -----------------------------------------------------------------
    @classmethod
    def zero(cls, n: int, mod_bits: int) -> "RingElement":
        torch = _torch()
        w = torch.zeros((words_for(mod_bits), n), dtype=torch.int32, device=_device())
        return cls(n, mod_bits, words=w)

    @classmethod
    def from_signed(cls, n: int, mod_bits: int, signed) -> "RingElement":
        """Element with the given signed coefficients; small values also get a compact view."""
        signed = list(signed)
        if len(signed) != n:
            raise ParameterError(f"expected {n} coefficients, got {len(signed)}")
        top = max((abs(c) for c in signed), default=0)
        el = cls(n, mod_bits, signed)
        cb = top.bit_length() + 1  # two's complement width holding every value
        if cb < mod_bits:
            el.compact_words = upload_words(ints_to_words(signed, cb))
            el.compact_bits = cb
        return el

    @classmethod
    def from_int64(cls, n: int, mod_bits: int, vals: np.ndarray) -> "RingElement":
        """Element with small signed coefficients given as an int64 array (|c| < 2^62),
        identical to from_signed on the same values but without Python ints."""
        vals = np.asarray(vals, dtype=np.int64)
        if vals.shape != (n,):
            raise ParameterError(f"expected {n} coefficients, got {vals.shape}")
        top = int(np.max(np.abs(vals))) if n else 0
        el = cls(n, mod_bits, words=upload_words(int64_to_words(vals, mod_bits)))
        cb = top.bit_length() + 1
        if cb < mod_bits:
            el.compact_words = upload_words(int64_to_words(vals, cb))
            el.compact_bits = cb
        return el

    @classmethod
    def from_words(cls, n: int, mod_bits: int, words) -> "RingElement":
        return cls(n, mod_bits, words=words)

    # -- host views ----------------------------------------------------------------------
    @property
    def coeffs(self) -> list[int]:
        return words_to_ints(download_words(self.words))

    def centered(self) -> list[int]:
        """Signed representatives in (-2^(bits-1), 2^(bits-1)] (ring.py:106-110)."""
        half = 1 << (self.mod_bits - 1)
        full = 1 << self.mod_bits
        return [c - full if c > half else c for c in self.coeffs]

    def numpy_words(self) -> np.ndarray:
        return download_words(self.words)

    # -- helpers ---------------------------------------------------------------------------
    def _require_same(self, other: "RingElement"):
        if self.n != other.n or self.mod_bits != other.mod_bits:
            raise ParameterError(
                f"ring mismatch: (n={self.n}, bits={self.mod_bits}) vs "
                f"(n={other.n}, bits={other.mod_bits})"
            )

    def _new(self, bits: int | None = None) -> "RingElement":
        bits = self.mod_bits if bits is None else bits
        return RingElement(self.n, bits, words=empty_words(bits, self.n))

    def operand(self, out_bits: int) -> _lib.Operand:
        """Narrowest legal view of this element for a product reduced mod 2^out_bits."""
        if self.compact_words is not None and out_bits <= self.mod_bits:
            return _lib.operand(self.compact_words, self.compact_bits, True)
        if out_bits <= self.mod_bits:
            return _lib.operand(self.words, self.mod_bits, True)   # centered representative
        return _lib.operand(self.words, self.mod_bits, False)      # canonical representative

    # -- arithmetic (ring.py:114-196) -----------------------------------------------------
    def add(self, other: "RingElement") -> "RingElement":
        self._require_same(other)
        out = self._new()
        ctx = _ctx(self.n)
        _lib.check(ctx.lib.hg_poly_add(ctx.handle, out.words.data_ptr(), self.words.data_ptr(),
                                       other.words.data_ptr(), self.mod_bits, ctx.stream()))
        return out

    @staticmethod
    def sum(elements: "list[RingElement]") -> "RingElement":
        """Exact sum mod 2^bits in one pass over the terms (== a fold of add)."""
        first = elements[0]
        for e in elements[1:]:
            first._require_same(e)
        out = first._new()
        ctx = _ctx(first.n)
        ptrs = (ctypes.c_void_p * len(elements))(*[e.words.data_ptr() for e in elements])
        _lib.check(ctx.lib.hg_poly_sum(ctx.handle, out.words.data_ptr(), ptrs, len(elements),
                                       first.mod_bits, ctx.stream()))
        return out

    def sub(self, other: "RingElement") -> "RingElement":
        self._require_same(other)
        out = self._new()
        ctx = _ctx(self.n)
        _lib.check(ctx.lib.hg_poly_sub(ctx.handle, out.words.data_ptr(), self.words.data_ptr(),
                                       other.words.data_ptr(), self.mod_bits, ctx.stream()))
        return out

    def neg(self) -> "RingElement":
        out = self._new()
        ctx = _ctx(self.n)
        _lib.check(ctx.lib.hg_poly_neg(ctx.handle, out.words.data_ptr(), self.words.data_ptr(),
                                       self.mod_bits, ctx.stream()))
        if self.compact_words is not None:
            pass  # negation of a compact view is not cached
        return out

    def scalar_mul(self, k: int) -> "RingElement":
        out = self._new()
        scalar_mul_into(out.words, self.words, self.mod_bits, k, self.n)
        return out

    def mul(self, other: "RingElement") -> "RingElement":
        self._require_same(other)
        return self.mul_mod(other, self.mod_bits)

    def mul_mod(self, other: "RingElement", out_bits: int) -> "RingElement":
        """Product reduced mod 2^out_bits; operands may carry different moduli (ring.py:145)."""
        if self.n != other.n:
            raise ParameterError("ring degree mismatch")
        out = self._new(out_bits)
        ctx = _ctx(self.n)
        _lib.check(ctx.lib.hg_poly_mul(ctx.handle, out.words.data_ptr(), out_bits,
                                       self.operand(out_bits), other.operand(out_bits),
                                       ctx.stream()))
        return out

    def automorphism(self, k: int) -> "RingElement":
        """x -> x^k for odd k (ring.py:152-166)."""
        if k % 2 == 0:
            raise ParameterError("automorphism exponent must be odd")
        out = self._new()
        ctx = _ctx(self.n)
        _lib.check(ctx.lib.hg_poly_automorphism(ctx.handle, out.words.data_ptr(),
                                                self.words.data_ptr(), self.mod_bits,
                                                int(k % (2 * self.n)), ctx.stream()))
        return out

    def reduce_to(self, bits: int) -> "RingElement":
        if bits > self.mod_bits:
            raise ParameterError(f"cannot reduce modulus upward ({self.mod_bits} -> {bits})")
        if bits == self.mod_bits:
            return self
        out = self._new(bits)
        ctx = _ctx(self.n)
        _lib.check(ctx.lib.hg_poly_reduce_to(ctx.handle, out.words.data_ptr(), bits,
                                             self.words.data_ptr(), self.mod_bits, ctx.stream()))
        if self.compact_words is not None and self.compact_bits < bits:
            out.compact_words, out.compact_bits = self.compact_words, self.compact_bits
        return out

    def lift_centered_to(self, bits: int) -> "RingElement":
        if bits < self.mod_bits:
            raise ParameterError("lift target smaller than current modulus")
        out = self._new(bits)
        ctx = _ctx(self.n)
        _lib.check(ctx.lib.hg_poly_lift_centered(ctx.handle, out.words.data_ptr(), bits,
                                                 self.words.data_ptr(), self.mod_bits,
                                                 ctx.stream()))
        if self.compact_words is not None:
            out.compact_words, out.compact_bits = self.compact_words, self.compact_bits
        return out

    def divide_round(self, shift: int, out_bits: int) -> "RingElement":
        """((c + 2^(shift-1)) >> shift) mod 2^out_bits (ring.py:184-196)."""
        out = self._new(out_bits)
        ctx = _ctx(self.n)
        _lib.check(ctx.lib.hg_poly_divide_round(ctx.handle, out.words.data_ptr(), out_bits,
                                                self.words.data_ptr(), self.mod_bits, shift,
                                                ctx.stream()))
        return out

    def to_float64(self) -> tuple[np.ndarray, float]:
        """float64 of the centered coefficients plus the power-of-two multiplier, exactly as
        encoding.py:93-105 computes them (Python float(int) rounding, the >960-bit shift),
        converted on the GPU; only the N doubles cross to the host."""
        torch = _torch()
        ctx = _ctx(self.n)
        out = torch.empty(self.n, dtype=torch.float64, device=self.words.device)
        aux = torch.empty(2, dtype=torch.int32, device=self.words.device)
        _lib.check(ctx.lib.hg_poly_to_double(ctx.handle, out.data_ptr(), aux.data_ptr(),
                                             self.words.data_ptr(), self.mod_bits, ctx.stream()))
        shift = int(aux[1].item())
        return out.cpu().numpy(), 2.0 ** min(shift, 300)

    # -- dunder ------------------------------------------------------------------------------
    def __eq__(self, other):
        if not isinstance(other, RingElement):
            return False
        if self.n != other.n or self.mod_bits != other.mod_bits:
            return False
        return bool(_torch().equal(self.words, other.words))

    def __hash__(self):
        return id(self)

    def __repr__(self):
        return f"RingElement(n={self.n}, mod_bits={self.mod_bits}, device)"


def scalar_mul_into(out_words, a_words, bits: int, k: int, n: int):
    """out = a * k mod 2^bits for an arbitrary Python integer k."""
    kk = k & ((1 << bits) - 1)
    kw = max(1, words_for(kk.bit_length()))
    arr = (_lib.ctypes.c_uint32 * kw)(*[(kk >> (32 * i)) & 0xFFFFFFFF for i in range(kw)])
    ctx = _ctx(n)
    if out_words.data_ptr() == a_words.data_ptr() and kw > 1:
        raise ParameterError("in-place scalar multiply needs a one-word scalar")
    _lib.check(ctx.lib.hg_poly_scalar_mul(ctx.handle, out_words.data_ptr(), a_words.data_ptr(),
                                          bits, arr, kw, ctx.stream()))


# -- coefficient samplers (host; restate ring.py:214-246 draw for draw) ------------------------

def sample_uniform(n: int, bits: int, rng: random.Random) -> list[int]:
    return [rng.getrandbits(bits) for _ in range(n)]


def _native_rng_call(rng: random.Random, fn):
    """Run a native sampler on rng's MT19937 state (getstate / setstate round trip): the
    Python generator then continues exactly after the native draws."""
    version, internal, gauss_next = rng.getstate()
    state = (ctypes.c_uint32 * 625)(*internal)
    g = ctypes.c_double(gauss_next if gauss_next is not None else 0.0)
    has = ctypes.c_int(0 if gauss_next is None else 1)
    out = fn(state, g, has)
    rng.setstate((version, tuple(state), g.value if has.value else None))
    return out


def _native_samplers() -> bool:
    """The host-side CPython-random replay in libhegwas_b200.so (hg_rng_*); HG_PY_SAMPLERS=1
    forces the Python loops (the two are bit-identical, tests/test_host.py)."""
    if os.environ.get("HG_PY_SAMPLERS"):
        return False
    try:
        return hasattr(_lib.load_library(), "hg_rng_ternary")
    except Exception:
        return False


def sample_gaussian_array(n: int, sigma: float, rng: random.Random) -> np.ndarray:
    """sample_gaussian as an int64 array (the native replay when available)."""
    if type(rng) is random.Random and n >= 64 and _native_samplers():
        buf = np.empty(n, dtype=np.int32)
        _native_rng_call(rng, lambda st, g, h: _lib.check(_lib.load_library().hg_rng_gaussian(
            st, ctypes.byref(g), ctypes.byref(h), n, float(sigma), buf.ctypes.data)))
        return buf.astype(np.int64)
    return np.asarray(sample_gaussian(n, sigma, rng), dtype=np.int64)


def sample_ternary_array(n: int, rng: random.Random) -> np.ndarray:
    """sample_ternary as an int64 array (the native replay when available)."""
    if type(rng) is random.Random and n >= 64 and _native_samplers():
        buf = np.empty(n, dtype=np.int8)
        _native_rng_call(rng, lambda st, g, h: _lib.check(_lib.load_library().hg_rng_ternary(
            st, n, buf.ctypes.data)))
        return buf.astype(np.int64)
    return np.asarray(sample_ternary(n, rng), dtype=np.int64)


def sample_gaussian(n: int, sigma: float, rng: random.Random) -> list[int]:
    """Rounded N(0, sigma^2), redrawing anything beyond 6 sigma."""
    if type(rng) is random.Random and n >= 64 and _native_samplers():
        return sample_gaussian_array(n, sigma, rng).tolist()
    cut = 6.0 * sigma
    out: list[int] = []
    gauss = rng.gauss
    while len(out) < n:
        x = gauss(0.0, sigma)
        if abs(x) <= cut:
            out.append(round(x))
    return out


def sample_hamming(n: int, h: int, rng: random.Random) -> list[int]:
    """Exactly h nonzero coefficients in {-1, +1} at distinct positions."""
    if h > n:
        raise ParameterError(f"Hamming weight {h} exceeds degree {n}")
    out = [0] * n
    for pos in rng.sample(range(n), h):
        out[pos] = 1 if rng.getrandbits(1) else -1
    return out


def sample_ternary(n: int, rng: random.Random) -> list[int]:
    """{-1, 0, 1} with probabilities 1/4, 1/2, 1/4 from two random bits each."""
    if type(rng) is random.Random and n >= 64 and _native_samplers():
        return sample_ternary_array(n, rng).tolist()
    table = (1, 0, 0, -1)
    return [table[rng.getrandbits(2)] for _ in range(n)]


def derive_rng(seed: int, *labels) -> random.Random:
    """Child generator for (seed, labels), seeded from a 64-bit blake2b digest."""
    tag = "/".join(str(x) for x in labels)
    digest = hashlib.blake2b(f"{seed}:{tag}".encode(), digest_size=8).digest()
    return random.Random(int.from_bytes(digest, "little"))


# -- device samplers (benchmark-scale inputs; not reference-reproducible) ---------------------

def small_element(n: int, bits: int, values) -> RingElement:
    """Element from small signed integers in a device tensor, with an 8-bit compact view."""
    torch = _torch()
    vals = values.to(torch.int64)
    w = words_for(bits)
    out = torch.empty((w, n), dtype=torch.int32, device=vals.device)
    low = vals & 0xFFFFFFFF
    out[0] = torch.where(low >= 2 ** 31, low - 2 ** 32, low).to(torch.int32)
    if w > 1:
        out[1:] = torch.where(vals < 0, -1, 0).to(torch.int32).unsqueeze(0)
    rem = bits & 31
    if rem:
        top = out[w - 1].to(torch.int64) & ((1 << rem) - 1)
        out[w - 1] = top.to(torch.int32)
    el = RingElement(n, bits, words=out)
    el.compact_words, el.compact_bits = (vals & 0xFF).to(torch.int32).unsqueeze(0), 8
    return el


def signed64_element(n: int, bits: int, values) -> RingElement:
    """Element from signed int64 coefficients (|c| < 2^62) held in a device tensor, with a
    64-bit (two-word) compact view: the device-side twin of RingElement.from_int64."""
    torch = _torch()
    vals = values.to(torch.int64)
    w = words_for(bits)
    if w < 2:
        raise ParameterError("signed64_element needs at least 64-bit moduli")
    out = torch.empty((w, n), dtype=torch.int32, device=vals.device)
    low = vals & 0xFFFFFFFF
    out[0] = torch.where(low >= 2 ** 31, low - 2 ** 32, low).to(torch.int32)
    out[1] = (vals >> 32).to(torch.int32)
    if w > 2:
        out[2:] = torch.where(vals < 0, -1, 0).to(torch.int32).unsqueeze(0)
    rem = bits & 31
    if rem:
        out[w - 1] = (out[w - 1].to(torch.int64) & ((1 << rem) - 1)).to(torch.int32)
    el = RingElement(n, bits, words=out)
    el.compact_words, el.compact_bits = out[:2].clone(), 64
    return el


def uniform_element(n: int, bits: int, gen) -> RingElement:
    """Uniform residues mod 2^bits drawn on the device."""
    torch = _torch()
    w = words_for(bits)
    out = torch.randint(-2 ** 31, 2 ** 31, (w, n), dtype=torch.int32, generator=gen, device=gen.device)
    rem = bits & 31
    if rem:
        out[w - 1] &= (1 << rem) - 1
    return RingElement(n, bits, words=out)


def device_ternary(n: int, gen):
    torch = _torch()
    t = torch.randint(0, 4, (n,), generator=gen, device=gen.device)
    return torch.where(t == 0, 1, torch.where(t == 3, -1, 0))


def device_gaussian(n: int, sigma: float, gen):
    """Rounded N(0, sigma^2) with the 6-sigma tail redrawn (same law as sample_gaussian)."""
    torch = _torch()
    x = torch.randn(n, generator=gen, device=gen.device, dtype=torch.float64) * sigma
    bad = x.abs() > 6.0 * sigma
    while bool(bad.any()):
        x[bad] = torch.randn(int(bad.sum()), generator=gen, device=gen.device, dtype=torch.float64) * sigma
        bad = x.abs() > 6.0 * sigma
    return torch.round(x).to(torch.int64)


def negacyclic_mul_host(a: list[int], b: list[int], n: int) -> list[int]:
    """Host negacyclic product for tiny rings (n <= 8), used only by client helpers."""
    out = [0] * n
    for i, x in enumerate(a):
        for j, y in enumerate(b):
            if i + j < n:
                out[i + j] += x * y
            else:
                out[i + j - n] -= x * y
    return out


__all__ = [
    "RingElement", "sample_uniform", "sample_gaussian", "sample_hamming", "sample_ternary",
    "derive_rng", "ints_to_words", "words_to_ints", "words_for", "math",
]
