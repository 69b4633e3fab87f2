"""Thin Python binding of the C ABI in include/dcopf_dual.h (ctypes).

Argument marshalling only: every step of the dual iteration runs in the
library's sm_100a kernels.  There is no CPU fallback -- if the shared library
or a CUDA device is missing, every call raises.

Arrays may be torch tensors (device or host) or numpy arrays (host); they are
passed to the library as raw pointers.  Per-instance arrays use the ABI's
instance-contiguous layout: load[n_bus][B], lambda[n_bus][B], ...
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

from . import _build

FORM_F2 = 0  # DCOPF_FORM_FLOW_BOX
FORM_F1 = 1  # DCOPF_FORM_LIMIT_ROWS
FORM_KVL = 2  # DCOPF_FORM_CYCLE (cluster and batched paths)
FORM_PTDF = 3  # DCOPF_FORM_PTDF: the paper's dense-PTDF Eq. 1, load-only batches (dense path)
PATH_AUTO, PATH_BATCHED, PATH_SINGLE, PATH_CLUSTER, PATH_DENSE = 0, 1, 2, 3, 4
INST_OK, INST_DIVERGED, INST_CONVERGED = 0, 1, 2
OPT_PLAIN, OPT_GDM, OPT_GDM_CLASSIC, OPT_ADAGRAD, OPT_ADAM = 0, 1, 2, 3, 4
ERRORS = {-1: "EINVAL", -2: "ETOPOLOGY", -3: "ECUDA", -4: "ENOMEM", -5: "ESTATE"}


class DcopfError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class NetworkDesc(ctypes.Structure):
    _fields_ = [("n_bus", ctypes.c_int32), ("n_branch", ctypes.c_int32), ("n_gen", ctypes.c_int32),
                ("ref_bus", ctypes.c_int32), ("br_from", ctypes.c_void_p), ("br_to", ctypes.c_void_p),
                ("br_b", ctypes.c_void_p), ("br_fmax", ctypes.c_void_p), ("theta_max", ctypes.c_void_p),
                ("gen_bus", ctypes.c_void_p), ("gen_pmin", ctypes.c_void_p), ("gen_pmax", ctypes.c_void_p),
                ("gen_c", ctypes.c_void_p), ("gen_a", ctypes.c_void_p), ("br_switchable", ctypes.c_void_p)]


class Options(ctypes.Structure):
    _fields_ = [("form", ctypes.c_int32), ("precision", ctypes.c_int32), ("device", ctypes.c_int32),
                ("path", ctypes.c_int32), ("single_max_batch", ctypes.c_int32),
                ("tile_parts", ctypes.c_int32), ("lane_instances", ctypes.c_int32), ("reserved", ctypes.c_int32 * 1)]


class Info(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int64), ("B_padded", ctypes.c_int64), ("path", ctypes.c_int32),
                ("form", ctypes.c_int32), ("n_bus", ctypes.c_int32), ("n_branch", ctypes.c_int32),
                ("n_gen", ctypes.c_int32), ("quadratic", ctypes.c_int32),
                ("alg_bytes_per_inst_iter", ctypes.c_int64), ("bandwidth", ctypes.c_int32),
                ("smem_bytes", ctypes.c_int32), ("threads_per_block", ctypes.c_int32),
                ("grid", ctypes.c_int32), ("launches_per_iter", ctypes.c_int32),
                ("state_on_chip", ctypes.c_int32), ("chunk", ctypes.c_int32),
                ("ring_bus", ctypes.c_int32), ("ring_branch", ctypes.c_int32), ("tile_width", ctypes.c_int32),
                ("copies_per_sweep", ctypes.c_int32), ("ring_life", ctypes.c_int32),
                ("cluster_size", ctypes.c_int32), ("tile_parts", ctypes.c_int32),
                ("lane_instances", ctypes.c_int32), ("halo_items", ctypes.c_int32),
                ("steps_per_sweep", ctypes.c_int32)]


class Optimizer(ctypes.Structure):
    _fields_ = [("variant", ctypes.c_int32), ("reserved", ctypes.c_int32), ("momentum", ctypes.c_double),
                ("beta1", ctypes.c_double), ("beta2", ctypes.c_double), ("epsilon", ctypes.c_double)]


SYMBOLS = ["dcopf_dual_create", "dcopf_dual_set_instance_batch", "dcopf_dual_iterate",
           "dcopf_dual_get_bound", "dcopf_dual_get_multipliers", "dcopf_dual_set_multipliers",
           "dcopf_dual_evaluate", "dcopf_dual_set_optimizer", "dcopf_dual_set_stop", "dcopf_dual_set_target", "dcopf_dual_get_first_hit", "dcopf_dual_get_info", "dcopf_dual_get_ptdf", "dcopf_dual_compact",
           "dcopf_dual_last_error", "dcopf_dual_destroy"]

_lib = None


def load_library(path: Optional[str] = None):
    """Load libdcopf_dual.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    path = path or os.environ.get("DCOPF_LIB") or _build.LIB  # DCOPF_LIB: A/B measurement of another build
    if not os.path.exists(path):
        raise ImportError(f"{path} not built; run __graft_entry__.build() (no CPU fallback exists)")
    lib = ctypes.CDLL(path)
    P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    lib.dcopf_dual_create.argtypes = [ctypes.POINTER(NetworkDesc), ctypes.POINTER(Options), ctypes.POINTER(P)]
    lib.dcopf_dual_set_instance_batch.argtypes = [P, I64, P, P, I32, P]
    lib.dcopf_dual_iterate.argtypes = [P, I64, P, P, P]
    lib.dcopf_dual_get_bound.argtypes = [P, P, P, P, P]
    lib.dcopf_dual_get_multipliers.argtypes = [P, P, P, P]
    lib.dcopf_dual_set_multipliers.argtypes = [P, P, P, P]
    lib.dcopf_dual_evaluate.argtypes = [P, P, P, P, P]
    if hasattr(lib, "dcopf_dual_set_optimizer"):
        lib.dcopf_dual_set_optimizer.argtypes = [P, ctypes.POINTER(Optimizer)]
    if hasattr(lib, "dcopf_dual_set_stop"):
        lib.dcopf_dual_set_stop.argtypes = [P, ctypes.c_double]
    if hasattr(lib, "dcopf_dual_set_target"):
        lib.dcopf_dual_set_target.argtypes = [P, P, P]
        lib.dcopf_dual_get_first_hit.argtypes = [P, P, P]
    lib.dcopf_dual_get_info.argtypes = [P, ctypes.POINTER(Info)]
    if hasattr(lib, "dcopf_dual_get_ptdf"):
        lib.dcopf_dual_get_ptdf.argtypes = [P, P, P]
    if hasattr(lib, "dcopf_dual_compact"):
        lib.dcopf_dual_compact.argtypes = [P, P, P, P]
    lib.dcopf_dual_last_error.argtypes = [P]
    lib.dcopf_dual_last_error.restype = ctypes.c_char_p
    lib.dcopf_dual_destroy.argtypes = [P]
    lib.dcopf_dual_destroy.restype = None
    for s in SYMBOLS[:-2]:
        if hasattr(lib, s):
            getattr(lib, s).restype = ctypes.c_int
    if path == _build.LIB:
        _lib = lib
    return lib


def _ptr(x):
    """Raw pointer of a torch tensor / numpy array / None (must be contiguous)."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        assert x.is_contiguous(), "tensor must be contiguous"
        return ctypes.c_void_p(x.data_ptr())
    assert isinstance(x, np.ndarray) and x.flags["C_CONTIGUOUS"]
    return x.ctypes.data_as(ctypes.c_void_p)


def _stream(s):
    if s is None:
        return None
    if hasattr(s, "cuda_stream"):
        return ctypes.c_void_p(s.cuda_stream)
    return ctypes.c_void_p(int(s))


class DcopfDual:
    """One library handle: a network + (after set_instance_batch) a batch."""

    def __init__(self, net, form: int = FORM_F2, device: int = 0, path: int = PATH_AUTO,
                 single_max_batch: int = 0, switchable=None, implied_theta: bool = False,
                 tile_parts: int = 0, lane_instances: int = 0):
        self.lib = load_library()
        self._keep = []
        k = lambda a, dt: (self._keep.append(np.ascontiguousarray(a, dtype=dt)) or self._keep[-1])
        d = NetworkDesc()
        d.n_bus, d.n_branch, d.n_gen, d.ref_bus = net.n_bus, net.n_branch, net.n_gen, net.ref_bus
        d.br_from = _ptr(k(net.br_from, np.int32))
        d.br_to = _ptr(k(net.br_to, np.int32))
        d.br_b = _ptr(k(net.br_b, np.float64))
        d.br_fmax = _ptr(k(net.br_fmax, np.float64))
        d.theta_max = None if implied_theta else _ptr(k(net.theta_max, np.float64))
        d.gen_bus = _ptr(k(net.gen_bus, np.int32))
        d.gen_pmin = _ptr(k(net.gen_pmin, np.float64))
        d.gen_pmax = _ptr(k(net.gen_pmax, np.float64))
        d.gen_c = _ptr(k(net.gen_c, np.float64))
        d.gen_a = None if net.gen_a is None else _ptr(k(net.gen_a, np.float64))
        d.br_switchable = None if switchable is None else _ptr(k(switchable, np.uint8))
        o = Options()
        o.form, o.precision, o.device, o.path, o.single_max_batch = form, 64, device, path, single_max_batch
        o.tile_parts, o.lane_instances = tile_parts, lane_instances
        h = ctypes.c_void_p()
        rc = self.lib.dcopf_dual_create(ctypes.byref(d), ctypes.byref(o), ctypes.byref(h))
        if rc != 0:
            raise DcopfError(rc, self.lib.dcopf_dual_last_error(None).decode())
        self.h = h
        self.net = net
        self.form = form
        self._keep = []

    # -- helpers --------------------------------------------------------------
    def _check(self, rc):
        if rc != 0:
            raise DcopfError(rc, self.lib.dcopf_dual_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            self.lib.dcopf_dual_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def n_branch_mult(self):
        if self.form == FORM_KVL:
            return self.net.n_branch - self.net.n_bus + 1
        return self.net.n_branch * (2 if self.form in (FORM_F1, FORM_PTDF) else 1)

    @property
    def n_lambda(self):
        """Rows of the lambda block: one per bus, one per instance for the PTDF form."""
        return 1 if self.form == FORM_PTDF else self.net.n_bus

    # -- ABI calls ------------------------------------------------------------
    def set_instance_batch(self, load, outages=None, stream=None):
        """load: [n_bus][B]; outages: [B][max_out] int32 (-1 padded) or None."""
        B = int(load.shape[1])
        max_out = 0 if outages is None else int(outages.shape[1])
        self._check(self.lib.dcopf_dual_set_instance_batch(self.h, B, _ptr(load), _ptr(outages), max_out,
                                                           _stream(stream)))
        self.B = B

    def iterate(self, K, alpha, history=None, stream=None):
        a = np.ascontiguousarray(alpha, dtype=np.float64)
        assert a.shape[0] >= K
        self._check(self.lib.dcopf_dual_iterate(self.h, int(K), _ptr(a), _ptr(history), _stream(stream)))

    def get_bound(self, bound=None, best=None, status=None, stream=None):
        self._check(self.lib.dcopf_dual_get_bound(self.h, _ptr(bound), _ptr(best), _ptr(status), _stream(stream)))

    def get_multipliers(self, lam=None, branch=None, stream=None):
        self._check(self.lib.dcopf_dual_get_multipliers(self.h, _ptr(lam), _ptr(branch), _stream(stream)))

    def set_multipliers(self, lam=None, branch=None, stream=None):
        self._check(self.lib.dcopf_dual_set_multipliers(self.h, _ptr(lam), _ptr(branch), _stream(stream)))

    def evaluate(self, value=None, grad_lam=None, grad_branch=None, stream=None):
        self._check(self.lib.dcopf_dual_evaluate(self.h, _ptr(value), _ptr(grad_lam), _ptr(grad_branch),
                                                 _stream(stream)))

    def set_optimizer(self, variant=OPT_PLAIN, momentum=0.0, beta1=0.0, beta2=0.0, epsilon=0.0):
        """Ascent-step variant (Algorithm 1); resets its state."""
        o = Optimizer()
        o.variant, o.momentum, o.beta1, o.beta2, o.epsilon = int(variant), momentum, beta1, beta2, epsilon
        self._check(self.lib.dcopf_dual_set_optimizer(self.h, ctypes.byref(o)))

    def set_stop(self, tol=0.0):
        """Algorithm 1's stopping rule |g_k - g_{k-1}| < tol per instance (0: off)."""
        self._check(self.lib.dcopf_dual_set_stop(self.h, float(tol)))

    def set_target(self, target=None, stream=None):
        """Per-instance time-to-gap thresholds [B] (None clears them)."""
        self._check(self.lib.dcopf_dual_set_target(self.h, _ptr(target), _stream(stream)))

    def get_first_hit(self, hit=None, stream=None):
        """[B] int64: first evaluation index whose running best >= target, or -1."""
        if hit is None:
            hit = np.empty(self.B, dtype=np.int64)
        self._check(self.lib.dcopf_dual_get_first_hit(self.h, _ptr(hit), _stream(stream)))
        return hit

    def compact(self, stream=None):
        """Drop the frozen (DIVERGED / CONVERGED) instances; returns the
        pre-compaction indices of the kept ones (their new order)."""
        kept = np.empty(self.B, dtype=np.int64)
        n = ctypes.c_int64(0)
        self._check(self.lib.dcopf_dual_compact(self.h, _ptr(kept), ctypes.byref(n), _stream(stream)))
        if 0 < n.value < self.B:
            self.B = int(n.value)
        return kept[:n.value].copy()

    def get_ptdf(self, Ha=None, stream=None):
        """PTDF form: the library's H_a [n_branch][n_bus]."""
        if Ha is None:
            Ha = np.empty((self.net.n_branch, self.net.n_bus))
        self._check(self.lib.dcopf_dual_get_ptdf(self.h, _ptr(Ha), _stream(stream)))
        return Ha

    def info(self) -> Info:
        inf = Info()
        self._check(self.lib.dcopf_dual_get_info(self.h, ctypes.byref(inf)))
        return inf

    # -- numpy conveniences (host buffers; the library does the copies) --------
    def results_numpy(self):
        B = self.B
        bound, best = np.empty(B), np.empty(B)
        status = np.empty(B, dtype=np.int32)
        self.get_bound(bound, best, status)
        lam = np.empty((self.n_lambda, B))
        br = np.empty((self.n_branch_mult, B))
        self.get_multipliers(lam, br)
        return bound, best, status, lam, br
