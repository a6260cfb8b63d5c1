"""ctypes marshalling for include/pmg_dg.h (argument conversion only; no arithmetic here)."""
import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PMG_LIB") or os.path.join(HERE, "libpmgdg.so")   # PMG_LIB: diagnostic builds only

GLL, GL = 0, 1
OVL_NODES, OVL_REL, OVL_MAXREL = 0, 1, 2
_CODES = {0: "PMG_OK", 1: "PMG_EINVAL", 2: "PMG_EDIM", 3: "PMG_ESINGULAR", 4: "PMG_ECUDA",
          5: "PMG_EWORKSPACE", 6: "PMG_EDIVERGED", 7: "PMG_EMAXIT", 8: "PMG_ESTATE"}

if not os.path.exists(LIB_PATH):
    raise ImportError("libpmgdg.so not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(no CPU fallback exists)")
lib = C.CDLL(LIB_PATH)

_vp, _dp, _ip, _i, _d, _ll, _sz = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int), C.c_int, \
    C.c_double, C.c_longlong, C.c_size_t
_sig = {
    "dg_setup": (_i, [_i, _i, _i, _d, _d, _d, _i, _i, _d, C.POINTER(_vp)]),
    "dg_schwarz_setup": (_i, [_vp, _i, _d, _i]),
    "dg_num_levels": (_i, [_vp]),
    "dg_ndofs": (_ll, [_vp, _i]),
    "dg_level_overlap": (_i, [_vp, _i, _ip, _ip]),
    "dg_get_table": (_i, [_vp, _i, _i, _i, _dp, _i]),
    "dg_workspace_bytes": (_sz, [_vp]),
    "dg_bind_workspace": (_i, [_vp, _vp, _sz, _vp]),
    "dg_apply": (_i, [_vp, _i, _vp, _vp, _vp]),
    "dg_residual": (_i, [_vp, _i, _vp, _vp, _vp, _vp]),
    "schwarz_smooth": (_i, [_vp, _i, _vp, _vp, _i, _vp]),
    "dg_schwarz_solve": (_i, [_vp, _i, _vp, _vp]),
    "dg_schwarz_fold": (_i, [_vp, _i, _vp, _i, _vp]),
    "dg_window_buffer": (_i, [_vp, _i, C.POINTER(_sz), C.POINTER(_ll)]),
    "dg_dot_range": (_i, [_vp, _vp, _vp, _ll, _dp, _vp]),
    "dg_axpby": (_i, [_vp, _vp, _d, _vp, _d, _ll, _vp]),
    "dg_prolongate_add": (_i, [_vp, _i, _vp, _vp, _vp]),
    "dg_restrict": (_i, [_vp, _i, _vp, _vp, _vp]),
    "dg_coarse_solve": (_i, [_vp, _vp, _vp, _vp]),
    "dg_set_schedule": (_i, [_vp, _ip, _ip]),
    "pmg_vcycle": (_i, [_vp, _vp, _vp, _vp]),
    "pcg_solve": (_i, [_vp, _vp, _vp, _d, _i, _ip, _dp, _vp]),
    "dg_dot": (_i, [_vp, _i, _vp, _vp, _dp, _vp]),
    "dg_project_mean": (_i, [_vp, _i, _vp, _vp]),
    "dg_rhs_sin": (_i, [_vp, _d, _d, _d, _d, _vp, _vp]),
    "dg_launch_count": (_ll, [_vp]),
    "dg_profile": (_i, [_vp, _i]),
    "dg_set_graphs": (_i, [_vp, _i]),
    "dg_set_colored": (_i, [_vp, _i]),
    "dg_profile_read": (_i, [_vp, _dp, C.POINTER(_ll), _i]),
    "pmg_fp64_peak": (_i, [_i, _dp, _vp]),
    "dg_last_error": (C.c_char_p, [_vp]),
    "dg_destroy": (None, [_vp]),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_sig)


class PMGError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("%s: %s" % (_CODES.get(code, code), msg))
        self.code = code


def _ptr(t):
    return C.c_void_p(t.data_ptr())


def _vec(t, n, what="vector"):
    """Pointer of a caller-owned device vector after the ABI's contract checks: CUDA, float64,
    contiguous, exactly n entries (a wrong tensor would otherwise read/write out of bounds)."""
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError("%s: expected a torch.Tensor" % what)
    if not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
        raise ValueError("%s: need a contiguous CUDA float64 tensor (got %s, %s, contiguous=%s)"
                         % (what, t.device, t.dtype, t.is_contiguous()))
    if t.numel() != n:
        raise ValueError("%s: %d entries, the level has %d DOF" % (what, t.numel(), n))
    return C.c_void_p(t.data_ptr())


def _stream():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


class DG:
    """One discretisation + multigrid hierarchy (dg_setup / dg_schwarz_setup / workspace)."""

    def __init__(self, ne, length, P, basis, penalty=2.0, overlap=None, bind=True):
        self._c = C.c_void_p()
        rc = lib.dg_setup(int(ne[0]), int(ne[1]), int(ne[2]), float(length[0]), float(length[1]),
                          float(length[2]), int(P), int(basis), float(penalty), C.byref(self._c))
        if rc:
            raise PMGError(rc, "dg_setup rejected its arguments")
        self.ne, self.length, self.P, self.basis = tuple(ne), tuple(length), P, basis
        self.ws = None
        if overlap is not None:
            self._check(lib.dg_schwarz_setup(self._c, int(overlap.mode), float(overlap.value),
                                             int(overlap.floor)))
        if bind:
            self.bind()

    def _check(self, rc):
        if rc:
            raise PMGError(rc, lib.dg_last_error(self._c).decode())
        return rc

    # ---- host queries
    @property
    def L(self):
        return lib.dg_num_levels(self._c) - 1

    def ndofs(self, level=None):
        return lib.dg_ndofs(self._c, self.L if level is None else level)

    def level_overlap(self, level):
        no = (C.c_int * 3)()
        m = (C.c_int * 3)()
        self._check(lib.dg_level_overlap(self._c, level, no, m))
        return list(no), list(m)

    def table(self, level, direction, which):
        import numpy as np
        cnt = lib.dg_get_table(self._c, level, direction, which, None, 0)
        if cnt < 0:
            raise PMGError(-cnt, "dg_get_table")
        out = np.zeros(max(cnt, 1))
        lib.dg_get_table(self._c, level, direction, which, out.ctypes.data_as(_dp), cnt)
        return out[:cnt]

    def launch_count(self):
        return lib.dg_launch_count(self._c)

    PROF_KINDS = ("traces", "apply", "fdm", "fold", "restrict", "prolong", "coarse", "vec")

    def set_colored(self, enable=True):
        self._check(lib.dg_set_colored(self._c, 1 if enable else 0))

    def set_graphs(self, enable=True):
        self._check(lib.dg_set_graphs(self._c, 1 if enable else 0))

    def profile(self, enable=True):
        self._check(lib.dg_profile(self._c, 1 if enable else 0))

    def profile_read(self, reset=True):
        """{(kind, level): (total_ms, launches)} accumulated by per-launch CUDA events."""
        ms = (C.c_double * 64)()
        cnt = (C.c_longlong * 64)()
        self._check(lib.dg_profile_read(self._c, ms, cnt, 1 if reset else 0))
        return {(self.PROF_KINDS[i // 8], i % 8): (ms[i], cnt[i]) for i in range(64) if cnt[i]}

    # ---- device
    def bind(self):
        import torch
        nbytes = lib.dg_workspace_bytes(self._c)
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        self._check(lib.dg_bind_workspace(self._c, _ptr(self.ws), nbytes, _stream()))

    def empty(self, level=None):
        import torch
        return torch.empty(self.ndofs(level), dtype=torch.float64, device="cuda")

    def apply(self, u, level=None, out=None):
        level = self.L if level is None else level
        n = self.ndofs(level)
        pu = _vec(u, n, "u")
        out = self.empty(level) if out is None else out
        self._check(lib.dg_apply(self._c, level, pu, _vec(out, n, "out"), _stream()))
        return out

    def residual(self, u, f, level=None, out=None):
        level = self.L if level is None else level
        n = self.ndofs(level)
        pu, pf = _vec(u, n, "u"), _vec(f, n, "f")
        out = self.empty(level) if out is None else out
        self._check(lib.dg_residual(self._c, level, pu, pf, _vec(out, n, "out"), _stream()))
        return out

    def schwarz_smooth(self, u, f, steps=1, level=None):
        level = self.L if level is None else level
        n = self.ndofs(level)
        self._check(lib.schwarz_smooth(self._c, level, _vec(u, n, "u"), _vec(f, n, "f"), int(steps), _stream()))
        return u

    def schwarz_solve(self, r, level=None):
        """First half of a Schwarz step: weighted subdomain solutions of r into the window buffer."""
        level = self.L if level is None else level
        self._check(lib.dg_schwarz_solve(self._c, level, _vec(r, self.ndofs(level), "r"), _stream()))

    def schwarz_fold(self, u, zero=False, level=None):
        """Second half: u (+)= deterministic sum of the weighted subdomain solutions."""
        level = self.L if level is None else level
        self._check(lib.dg_schwarz_fold(self._c, level, _vec(u, self.ndofs(level), "u"), 1 if zero else 0,
                                        _stream()))
        return u

    def window_buffer(self, level=None):
        """Zero-copy float64 view of level l's window buffer inside the workspace
        (subdomains in element order, dg_window_buffer doubles each)."""
        import torch
        level = self.L if level is None else level
        off, per = _sz(0), _ll(0)
        self._check(lib.dg_window_buffer(self._c, level, C.byref(off), C.byref(per)))
        ne = self.ne[0] * self.ne[1] * self.ne[2]
        nbytes = 8 * per.value * ne
        return self.ws[off.value: off.value + nbytes].view(torch.float64), per.value

    def dot_range(self, x, y, count):
        """<x, y> over the first `count` entries of two contiguous CUDA float64 tensors."""
        import torch
        for t in (x, y):
            if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()
                    and t.numel() >= count):
                raise ValueError("dot_range: need contiguous CUDA float64 tensors with >= count entries")
        v = C.c_double(0)
        self._check(lib.dg_dot_range(self._c, _ptr(x), _ptr(y), int(count), C.byref(v), _stream()))
        return v.value

    def axpby(self, y, a, x, b=1.0):
        """y = a x + b y (same-size contiguous CUDA float64 tensors)."""
        import torch
        for t in (x, y):
            if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
                raise ValueError("axpby: need contiguous CUDA float64 tensors")
        if x.numel() != y.numel():
            raise ValueError("axpby: size mismatch")
        self._check(lib.dg_axpby(self._c, _ptr(y), float(a), _ptr(x), float(b), y.numel(), _stream()))
        return y

    def prolongate_add(self, uc, uf, level):
        self._check(lib.dg_prolongate_add(self._c, level, _vec(uc, self.ndofs(level - 1), "uc"),
                                          _vec(uf, self.ndofs(level), "uf"), _stream()))
        return uf

    def restrict(self, rf, level, out=None):
        prf = _vec(rf, self.ndofs(level), "rf")
        out = self.empty(level - 1) if out is None else out
        self._check(lib.dg_restrict(self._c, level, prf, _vec(out, self.ndofs(level - 1), "out"), _stream()))
        return out

    def coarse_solve(self, f0, out=None):
        n = self.ndofs(0)
        pf = _vec(f0, n, "f0")
        out = self.empty(0) if out is None else out
        self._check(lib.dg_coarse_solve(self._c, pf, _vec(out, n, "out"), _stream()))
        return out

    def set_schedule(self, nu1, nu2):
        if len(nu1) != self.L + 1 or len(nu2) != self.L + 1:
            raise ValueError("set_schedule: nu1, nu2 need L+1 = %d entries" % (self.L + 1))
        a = (C.c_int * len(nu1))(*nu1)
        b = (C.c_int * len(nu2))(*nu2)
        self._check(lib.dg_set_schedule(self._c, a, b))

    def pmg_vcycle(self, u, f):
        n = self.ndofs()
        self._check(lib.pmg_vcycle(self._c, _vec(u, n, "u"), _vec(f, n, "f"), _stream()))
        return u

    def pcg_solve(self, u, f, rtol=1e-10, maxit=100):
        import numpy as np
        it = C.c_int(0)
        hist = np.zeros(maxit + 1)
        n = self.ndofs()
        rc = lib.pcg_solve(self._c, _vec(u, n, "u"), _vec(f, n, "f"), float(rtol), int(maxit), C.byref(it),
                           hist.ctypes.data_as(_dp), _stream())
        if rc and rc != 7:
            self._check(rc)
        return u, hist[: it.value + 1], rc == 0

    def dot(self, x, y, level=None):
        level = self.L if level is None else level
        v = C.c_double(0)
        n = self.ndofs(level)
        self._check(lib.dg_dot(self._c, level, _vec(x, n, "x"), _vec(y, n, "y"), C.byref(v), _stream()))
        return v.value

    def project_mean(self, v, level=None):
        level = self.L if level is None else level
        self._check(lib.dg_project_mean(self._c, level, _vec(v, self.ndofs(level), "v"), _stream()))
        return v

    def rhs_sin(self, amp, kx, ky, kz, out=None):
        out = self.empty() if out is None else out
        self._check(lib.dg_rhs_sin(self._c, float(amp), float(kx), float(ky), float(kz), _vec(out, self.ndofs(), "out"),
                                   _stream()))
        return out

    def close(self):
        if self._c:
            lib.dg_destroy(self._c)
            self._c = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fp64_peak_tflops(use_dmma=False):
    """Measured FP64 DFMA (or DMMA) throughput of the current GPU (pmg_fp64_peak)."""
    v = C.c_double(0)
    rc = lib.pmg_fp64_peak(1 if use_dmma else 0, C.byref(v), _stream())
    if rc:
        raise PMGError(rc, "pmg_fp64_peak failed")
    return v.value


def dg_setup(ne, length, P, basis, penalty=2.0, overlap=None, bind=True):
    """Python spelling of the C entry point dg_setup (+ dg_schwarz_setup when overlap is given)."""
    return DG(ne, length, P, basis, penalty, overlap, bind)
