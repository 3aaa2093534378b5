"""ctypes binding of libhegwas_b200.so (the C-ABI in include/hegwas_b200.h).

There is no CPU fallback: if the shared library is missing or no CUDA device is
present, every device operation raises.  Build the library with
``python -c "import __graft_entry__ as g; g.build()"`` (or ``make -C
paper_1902_04303_b200/csrc``).
"""
from __future__ import annotations

import ctypes
import os
import threading

from .errors import HegwasError, ParameterError

_HERE = os.path.dirname(os.path.abspath(__file__))
# HG_LIB_PATH: load an alternative build of the same C-ABI (kernel experiments)
LIB_PATH = os.environ.get("HG_LIB_PATH") or os.path.join(_HERE, "libhegwas_b200.so")

HG_OK = 0
HG_EINVAL = 1
HG_ENOMEM = 2
HG_ECUDA = 3
HG_ERANGE = 4


class DeviceError(HegwasError):
    """CUDA failure or missing native library (never silently falls back)."""


class Operand(ctypes.Structure):
    _fields_ = [("words", ctypes.c_void_p), ("bits", ctypes.c_int32), ("signed_rep", ctypes.c_int32)]


_u32p = ctypes.POINTER(ctypes.c_uint32)
_vp = ctypes.c_void_p
_i = ctypes.c_int
_i64 = ctypes.c_int64

# name -> (restype, argtypes)
SIGNATURES = {
    "hg_last_error": (ctypes.c_char_p, []),
    "hg_version": (_i, []),
    "hg_ctx_create": (_i, [_i, _i, ctypes.POINTER(_vp)]),
    "hg_ctx_destroy": (_i, [_vp]),
    "hg_ctx_max_product_bits": (_i, [_vp]),
    "hg_ctx_num_primes": (_i, [_vp]),
    "hg_ctx_primes": (_i, [_vp, _u32p]),
    "hg_sync": (_i, [_vp, _vp]),
    "hg_poly_add": (_i, [_vp, _vp, _vp, _vp, _i, _vp]),
    "hg_poly_sub": (_i, [_vp, _vp, _vp, _vp, _i, _vp]),
    "hg_poly_neg": (_i, [_vp, _vp, _vp, _i, _vp]),
    "hg_poly_scalar_mul": (_i, [_vp, _vp, _vp, _i, _u32p, _i, _vp]),
    "hg_poly_reduce_to": (_i, [_vp, _vp, _i, _vp, _i, _vp]),
    "hg_poly_lift_centered": (_i, [_vp, _vp, _i, _vp, _i, _vp]),
    "hg_poly_divide_round": (_i, [_vp, _vp, _i, _vp, _i, _i, _vp]),
    "hg_poly_automorphism": (_i, [_vp, _vp, _vp, _i, _i64, _vp]),
    "hg_poly_to_double": (_i, [_vp, _vp, _vp, _vp, _i, _vp]),
    "hg_poly_mul": (_i, [_vp, _vp, _i, Operand, Operand, _vp]),
    "hg_poly_tensor": (_i, [_vp, _vp, _vp, _vp, _i, Operand, Operand, Operand, Operand, _vp]),
    "hg_key_prepare": (_i, [_vp, _vp, _vp, _i, _i, _i, _vp, ctypes.POINTER(_vp)]),
    "hg_key_destroy": (_i, [_vp]),
    "hg_key_release": (_i, [_vp, _vp]),
    "hg_ctprep_release": (_i, [_vp, _vp]),
    "hg_key_device_bytes": (ctypes.c_size_t, [_vp]),
    "hg_keyswitch": (_i, [_vp, _vp, _vp, _i64, _vp, _vp, _vp]),
    "hg_ct_mult": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _i, _i, _vp, _vp, _vp]),
    "hg_ct_automorph": (_i, [_vp, _vp, _vp, _vp, _i, _i64, _vp, _vp, _vp]),
    "hg_ct_automorph_batch": (_i, [_vp, _vp, _i, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _i, _i64,
                                   ctypes.POINTER(_vp), ctypes.POINTER(_vp), _vp]),
"hg_ct_rotate_add_batch": (_i, [_vp, _vp, _i, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _i, _i64,
                                   ctypes.POINTER(_vp), ctypes.POINTER(_vp), _vp]),
    "hg_ct_prepare": (_i, [_vp, _vp, _vp, _i, _vp, ctypes.POINTER(_vp)]),
    "hg_ct_mult_batch": (_i, [_vp, _vp, _i, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                              ctypes.POINTER(_vp), _i, _i, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _vp]),
    "hg_ct_mult_prepared_batch": (_i, [_vp, _vp, _i, ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                       ctypes.POINTER(_vp), _i, _i, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _vp]),
    "hg_ct_prepare_sum": (_i, [_vp, _vp, _vp, _i, _i, _vp, ctypes.POINTER(_vp)]),
    "hg_ct_inner_prepared": (_i, [_vp, _vp, _i, _i, ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                  ctypes.POINTER(_vp), _i, _i, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _vp]),
    "hg_ctprep_destroy": (_i, [_vp]),
    "hg_ctprep_device_bytes": (ctypes.c_size_t, [_vp]),
    "hg_ct_mult_prepared": (_i, [_vp, _vp, _vp, _vp, _vp, _i, _i, _vp, _vp, _vp]),
    "hg_ct_mult_plain_many": (_i, [_vp, _vp, _vp, _i, _i, ctypes.POINTER(Operand), _i, ctypes.POINTER(_vp),
                                   ctypes.POINTER(_vp), _vp]),
    "hg_ct_mult_plain_batch": (_i, [_vp, _i, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _i, Operand, _i,
                                    ctypes.POINTER(_vp), ctypes.POINTER(_vp), _vp]),
    "hg_ct_rescale_batch": (_i, [_vp, _i, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _i, _i,
                                 ctypes.POINTER(_vp), ctypes.POINTER(_vp), _vp]),
    "hg_ct_add_batch": (_i, [_vp, _i, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                             ctypes.POINTER(_vp), _i, _i, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _vp]),
    "hg_ct_mult_const_rescale_batch": (_i, [_vp, _i, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _i, _i64, _i,
                                            ctypes.POINTER(_vp), ctypes.POINTER(_vp), _vp]),
    "hg_ntt_forward": (_i, [_vp, _vp, _i, _i, _vp]),
    "hg_ntt_inverse": (_i, [_vp, _vp, _i, _i, _vp]),
    "hg_set_ntt_variant": (_i, [_vp, _i]),
    "hg_bench_modmul": (_i, [_vp, _i, _vp, ctypes.POINTER(ctypes.c_double), _vp]),
    "hg_bench_mac": (_i, [_vp, _i, _vp, ctypes.POINTER(ctypes.c_double), _vp]),
    "hg_launch_count": (ctypes.c_longlong, [_vp]),
    "hg_set_kernel_timing": (_i, [_vp, _i]),
    "hg_poly_sum": (_i, [_vp, _vp, ctypes.POINTER(ctypes.c_void_p), _i, _i, _vp]),
    "hg_rng_ternary": (_i, [_vp, _i, _vp]),
    "hg_rng_gaussian": (_i, [_vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_i), _i, ctypes.c_double, _vp]),
    "hg_pool_reserve": (_i, [_vp, ctypes.c_size_t, _vp]),
    "hg_pool_bytes": (ctypes.c_size_t, [_vp, _i]),
    "hg_pool_trim": (ctypes.c_size_t, [_vp]),
    "hg_kernel_stats": (_i, [_vp, _i, ctypes.POINTER(ctypes.c_double),
                             ctypes.POINTER(ctypes.c_longlong), ctypes.POINTER(ctypes.c_double)]),
}

KERNEL_KINDS = {"crt": 0, "modup": 1, "ntt": 2, "pointwise": 3, "elementwise": 4}

_lib = None
_lock = threading.RLock()


def load_library(path: str = LIB_PATH):
    """Load and type the shared library (no CUDA calls are made)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise DeviceError(
                f"native library {path} not built; run __graft_entry__.build() "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int):
    if rc == HG_OK:
        return
    msg = load_library().hg_last_error().decode(errors="replace")
    if rc in (HG_EINVAL, HG_ERANGE):
        raise ParameterError(msg)
    raise DeviceError(f"native error {rc}: {msg}")


def check_alloc(call, evict=None):
    """check(call()) for an entry point that allocates from the device arena.  On HG_ENOMEM
    the device memory torch's caching allocator holds unused is handed back (and, failing
    that, ``evict()`` drops cached prepared keys) before one retry: the two allocators
    share the HBM and neither can take memory the other has cached."""
    rc = call()
    if rc == HG_ENOMEM:
        release_device_memory()
        rc = call()
        if rc == HG_ENOMEM and evict is not None:
            evict()
            torch.cuda.synchronize()
            rc = call()
    check(rc)


def _is_oom(rc: int) -> bool:
    if rc == HG_ENOMEM:
        return True
    return rc == HG_ECUDA and b"out of memory" in load_library().hg_last_error()


def call(fn, *args):
    """check(fn(*args)) for a product entry point whose scratch comes from the library's
    stream-ordered pool: on out-of-memory the caches torch and the library hold are handed
    back and the call is repeated once (the entry points never write their inputs, so a
    repeat recomputes every output from unchanged operands)."""
    rc = fn(*args)
    if rc != HG_OK and _is_oom(rc):
        global OOM_RETRIES
        OOM_RETRIES += 1
        release_device_memory()
        rc = fn(*args)
    check(rc)


OOM_RETRIES = 0   # library-scratch out-of-memory retries so far (diagnostics)


def operand(words, bits: int, signed: bool) -> Operand:
    return Operand(ctypes.c_void_p(words.data_ptr()), int(bits), 1 if signed else 0)


class Context:
    """One native context per (log_n, device): prime basis, twiddles, CRT tables."""

    def __init__(self, log_n: int, device: int):
        import torch

        if not torch.cuda.is_available():
            raise DeviceError("no CUDA device: the B200 evaluator has no CPU fallback")
        self.lib = load_library()
        self.log_n = log_n
        self.device = device
        handle = ctypes.c_void_p()
        with torch.cuda.device(device):
            check(self.lib.hg_ctx_create(log_n, device, ctypes.byref(handle)))
        self.handle = handle

    def stream(self):
        import torch

        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def compute_stream(self):
        """The device's default torch stream, where this package issues its compute (the side
        streams only copy): stream-ordered frees are ordered after it."""
        import torch

        return ctypes.c_void_p(torch.cuda.default_stream(self.device).cuda_stream)

    def primes(self) -> list[int]:
        n = self.lib.hg_ctx_num_primes(self.handle)
        arr = (ctypes.c_uint32 * n)()
        check(self.lib.hg_ctx_primes(self.handle, arr))
        return list(arr)

    def launches(self) -> int:
        return int(self.lib.hg_launch_count(self.handle))

    def set_kernel_timing(self, enabled: bool, kinds=None):
        """Bracket launches with CUDA events: every class, or only `kinds` (names)."""
        if not enabled:
            code = 0
        elif kinds is None:
            code = 1
        else:
            code = sum(1 << KERNEL_KINDS[k] for k in kinds) << 1
        check(self.lib.hg_set_kernel_timing(self.handle, code))

    def pool_reserve(self, nbytes: int) -> None:
        """Reserve one more device-arena slab of nbytes (hg_pool_reserve)."""
        check(self.lib.hg_pool_reserve(self.handle, int(nbytes), self.stream()))

    def pool_trim(self) -> int:
        return int(self.lib.hg_pool_trim(self.handle))

    def pool_bytes(self, in_use: bool = False) -> int:
        return int(self.lib.hg_pool_bytes(self.handle, 1 if in_use else 0))

    def kernel_stats(self, kind: str) -> dict:
        """{'ms', 'launches', 'work'} of the events recorded since timing was enabled."""
        ms, n, work = ctypes.c_double(), ctypes.c_longlong(), ctypes.c_double()
        check(self.lib.hg_kernel_stats(self.handle, KERNEL_KINDS[kind], ctypes.byref(ms),
                                       ctypes.byref(n), ctypes.byref(work)))
        return {"ms": ms.value, "launches": n.value, "work": work.value}

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            if self.handle:
                self.lib.hg_ctx_destroy(self.handle)
        except Exception:
            pass


_contexts: dict[tuple[int, int], Context] = {}


def release_device_memory() -> int:
    """Hand back device memory held only by caches: prepared keys of switching keys that no
    longer exist, arena slabs with no live object, torch's unused cached blocks.  Called on
    an allocation failure before one retry (the library arena and torch's caching allocator
    share the HBM and neither can take memory the other holds)."""
    import torch

    freed = 0
    try:
        from .ckks import KEY_CACHE

        KEY_CACHE.purge_dead()
    except Exception:
        pass
    torch.cuda.synchronize()
    for ctx in list(_contexts.values()):
        freed += ctx.pool_trim()
    torch.cuda.empty_cache()
    return freed


def get_context(log_n: int, device: int | None = None) -> Context:
    import torch

    if device is None:
        device = torch.cuda.current_device() if torch.cuda.is_available() else 0
    key = (log_n, device)
    ctx = _contexts.get(key)
    if ctx is None:
        with _lock:
            ctx = _contexts.get(key)
            if ctx is None:
                ctx = Context(log_n, device)
                _contexts[key] = ctx
    return ctx


def total_launches() -> int:
    return sum(c.launches() for c in _contexts.values())
