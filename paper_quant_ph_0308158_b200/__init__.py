"""B200-native hot path of Burger's permutation-map quantum-circuit simulator
(arXiv quant-ph/0308158).

A thin ctypes binding over ``libqsim.so`` (C ABI in ``include/qsim.h``):
argument marshalling only -- every step of the path (the address walk and the
gather) runs in the sm_100a kernels under ``csrc/``.  PyTorch supplies device
memory and streams.  There is no CPU fallback: if the library is missing the
import fails.

    import paper_quant_ph_0308158_b200 as qsim
    qsim.build_map(gates, M, perm)            # perm[i] = f_1(...f_n(i))
    qsim.apply_map(perm, M, k1, k2)           # k2[i] = k1[perm[i]]
    qsim.run_fused(gates, M, k1, k2)          # same k2, no perm buffer

``gates`` is a uint8 array of shape (n, 4): (kind, target, c0, c1), kind
0 NOT / 1 CNOT / 2 CCNOT, 0-based bits (bit b = a(b+1), a(1) the LSB),
row 0 = Step 1 (applied first).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libqsim.so")

OK, EINVAL, ERANGE, EBIT, ECAP, EALIAS, ECUDA = 0, -1, -2, -3, -4, -5, -6
C64, C128 = 0, 1
WALK_AUTO, WALK_PER_LANE, WALK_BITSLICED, WALK_JIT = 0, 1, 2, 3
# gate kinds (include/qsim.h): toggles, phase steps (reading R17), SWAP
NOT, CNOT, CCNOT, Z, CZ, CCZ, SWAP = 0, 1, 2, 3, 4, 5, 6
MAX_GATES = 4096
MATERIALISED, FUSED = 0, 1
TUNE_MEASURE, TUNE_PATIENT = 1, 2      # qsim_plan_tune_ex search effort
TUNE_APPLY = 0x100                     # | effort: tune the planned apply (perm built first)


class QsimError(RuntimeError):
    def __init__(self, code: int, where: str):
        lib = _lib
        msg = lib.qsim_strerror(code).decode()
        if code == ECUDA:
            msg += ": " + lib.qsim_last_error().decode()
        super().__init__(f"{where}: {msg} (status {code})")
        self.code = code


WORKSPACE_BYTES = 256
PLAN_SPLIT = 4                         # qsim_plan.flags bit 2 (QSIM_PLAN_SPLIT)


class Plan(ctypes.Structure):
    """qsim_plan (include/qsim.h): traversal order of the gather."""
    _fields_ = [("M", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("chunk_log2", ctypes.c_uint32), ("blocks_per_sm", ctypes.c_int32),
                ("flags", ctypes.c_uint32), ("ilp", ctypes.c_uint16),
                ("cta_threads", ctypes.c_uint16), ("fused_chunk_log2", ctypes.c_uint16),
                ("reserved_spread", ctypes.c_uint16),
                ("sigma", ctypes.c_uint8 * 32), ("change_freq", ctypes.c_float * 32),
                ("tile_log2", ctypes.c_uint8), ("tile_reserved", ctypes.c_uint8 * 3),
                ("tile_contained", ctypes.c_float)]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    vp, u64, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int32
    sig = {
        "qsim_build_map": [vp, i32, i32, vp, vp],
        "qsim_build_map_range": [vp, i32, i32, u64, u64, vp, vp],
        "qsim_build_map_ex": [vp, i32, i32, u64, u64, vp, i32, vp],
        "qsim_apply_map": [vp, i32, i32, vp, vp, vp],
        "qsim_apply_map_range": [vp, u64, i32, i32, vp, vp, vp],
        "qsim_run_fused": [vp, i32, i32, i32, vp, vp, vp],
        "qsim_run_fused_range": [vp, i32, i32, i32, u64, u64, vp, vp, vp],
        "qsim_run_fused_ex": [vp, i32, i32, i32, u64, u64, vp, vp, i32, vp],
        "qsim_run_host": [vp, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp],
    }
    sig["qsim_build_map_signed"] = [vp, i32, i32, u64, u64, vp, vp, vp]
    sig["qsim_run_host_batch"] = [vp, i32, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp]
    sig["qsim_graph_create"] = [ctypes.POINTER(Plan), vp, i32, i32, vp, vp, vp, vp, i32,
                                ctypes.POINTER(vp)]
    sig["qsim_graph_launch"] = [vp, vp]
    sig["qsim_plan_tune"] = [ctypes.POINTER(Plan), vp, i32, vp, vp, vp, vp, vp,
                             ctypes.POINTER(i32)]
    sig["qsim_plan_tune_ex"] = [ctypes.POINTER(Plan), vp, i32, vp, vp, vp, vp, vp, i32,
                                ctypes.POINTER(i32)]
    sig["qsim_graph_destroy"] = [vp]
    sig["qsim_apply_map_signed"] = [vp, vp, u64, i32, i32, vp, vp, vp]
    sig["qsim_plan_create"] = [vp, i32, i32, i32, ctypes.POINTER(Plan)]
    sig["qsim_apply_map_planned"] = [ctypes.POINTER(Plan), vp, vp, vp, vp, vp]
    sig["qsim_run_fused_planned"] = [ctypes.POINTER(Plan), vp, i32, vp, vp, vp, vp]
    sig["qsim_map_gather_planned"] = [ctypes.POINTER(Plan), vp, i32, vp, vp, vp, vp, vp]
    sig["qsim_jit_check_compile"] = [vp, i32, i32]
    sig["qsim_jit_check_compile_kron"] = [vp, i32, i32, i32]
    sig["qsim_run_fused_kron"] = [vp, i32, i32, i32, vp, u64, u64, vp, i32, vp]
    sig["qsim_jit_check_compile_planned"] = [ctypes.POINTER(Plan), vp, i32]
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    lib.qsim_strerror.argtypes = [i32]
    lib.qsim_strerror.restype = ctypes.c_char_p
    lib.qsim_last_error.argtypes = []
    lib.qsim_last_error.restype = ctypes.c_char_p
    lib.qsim_abi_version.restype = i32
    lib.qsim_jit_status.restype = ctypes.c_char_p
    lib.qsim_jit_last_compile_ms.restype = ctypes.c_double
    lib.qsim_last_launch_count.restype = i32
    lib.qsim_last_kernel.restype = ctypes.c_char_p
    return lib


_lib = _load()


def lib() -> ctypes.CDLL:
    return _lib


# ------------------------------------------------------------------ marshalling
def _gates(gates):
    g = np.ascontiguousarray(np.asarray(gates, dtype=np.uint8).reshape(-1, 4))
    return g, (g.ctypes.data if g.shape[0] else None), int(g.shape[0])


def _ptr(x) -> int | None:
    """Device or host address of a torch tensor / numpy array / int."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()                     # torch.Tensor


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _dtype_code(x) -> int:
    if isinstance(x, int):
        return x
    s = str(getattr(x, "dtype", x))
    if "complex64" in s or s == "c64":
        return C64
    if "complex128" in s or s == "c128":
        return C128
    raise TypeError(f"state dtype must be complex64 or complex128, got {s}")


def _check(rc: int, where: str) -> None:
    if rc != OK:
        raise QsimError(rc, where)


_ELEM = {C64: 8, C128: 16}


def _need(x, nbytes: int, what: str, device: bool = True) -> None:
    """Argument check before the C call (the ABI cannot see sizes): a torch
    tensor must be on CUDA (device buffers) and hold at least nbytes; a numpy
    array must hold at least nbytes.  Raw integer addresses are passed on."""
    if x is None or isinstance(x, int):
        return
    if isinstance(x, np.ndarray):
        have = x.nbytes
    else:
        if device and not x.is_cuda:
            raise ValueError(f"{what} must be a CUDA tensor (got device {x.device})")
        have = x.numel() * x.element_size()
    if have < nbytes:
        raise ValueError(f"{what} holds {have} bytes, the call needs {nbytes}")


def _tensor_dtype(x):
    """C64 / C128 from a complex tensor or array, else None (raw bytes)."""
    s = str(getattr(x, "dtype", ""))
    if "complex64" in s:
        return C64
    if "complex128" in s:
        return C128
    return None


# ---------------------------------------------------------------------- calls
def build_map(gates, M: int, perm, stream=None) -> None:
    g, gp, n = _gates(gates)
    if 1 <= M <= 32:
        _need(perm, 4 << M, "perm")
    _check(_lib.qsim_build_map(gp, n, M, _ptr(perm), _stream(stream)), "qsim_build_map")


def build_map_range(gates, M: int, start: int, count: int, perm_out, stream=None,
                    walk: int = WALK_AUTO) -> None:
    g, gp, n = _gates(gates)
    _need(perm_out, 4 * count, "perm_out")
    _check(_lib.qsim_build_map_ex(gp, n, M, start, count, _ptr(perm_out), walk,
                                  _stream(stream)), "qsim_build_map_ex")


def build_map_signed(gates, M: int, start: int, count: int, perm_out, signs, stream=None) -> None:
    """Phased permutation (Z / CZ / CCZ / SWAP steps allowed): perm_out and the
    row values as a bitmap, bit r % 32 of signs[r // 32] = 1 for -1."""
    g, gp, n = _gates(gates)
    _check(_lib.qsim_build_map_signed(gp, n, M, start, count, _ptr(perm_out), _ptr(signs),
                                      _stream(stream)), "qsim_build_map_signed")


def apply_map_signed(perm_in, signs, count: int, M: int, k1, k2_out, stream=None,
                     dtype=None) -> None:
    code = _dtype_code(k1 if dtype is None else dtype)
    _check(_lib.qsim_apply_map_signed(_ptr(perm_in), _ptr(signs), count, M, code, _ptr(k1),
                                      _ptr(k2_out), _stream(stream)), "qsim_apply_map_signed")


def apply_map(perm, M: int, k1, k2, stream=None, dtype=None) -> None:
    code = _dtype_code(k1 if dtype is None else dtype)
    if 1 <= M <= 32 and code in _ELEM:
        _need(perm, 4 << M, "perm")
        _need(k1, _ELEM[code] << M, "k1")
        _need(k2, _ELEM[code] << M, "k2")
    _check(_lib.qsim_apply_map(_ptr(perm), M, code, _ptr(k1), _ptr(k2), _stream(stream)),
           "qsim_apply_map")


def apply_map_range(perm_in, count: int, M: int, k1, k2_out, stream=None, dtype=None) -> None:
    code = _dtype_code(k1 if dtype is None else dtype)
    _check(_lib.qsim_apply_map_range(_ptr(perm_in), count, M, code, _ptr(k1), _ptr(k2_out),
                                     _stream(stream)), "qsim_apply_map_range")


def run_fused(gates, M: int, k1, k2, stream=None, dtype=None) -> None:
    g, gp, n = _gates(gates)
    code = _dtype_code(k1 if dtype is None else dtype)
    if 1 <= M <= 32 and code in _ELEM:
        _need(k1, _ELEM[code] << M, "k1")
        _need(k2, _ELEM[code] << M, "k2")
    _check(_lib.qsim_run_fused(gp, n, M, code, _ptr(k1), _ptr(k2), _stream(stream)),
           "qsim_run_fused")


def run_fused_range(gates, M: int, start: int, count: int, k1, k2_out, stream=None,
                    dtype=None, walk: int = WALK_AUTO) -> None:
    g, gp, n = _gates(gates)
    code = _dtype_code(k1 if dtype is None else dtype)
    _check(_lib.qsim_run_fused_ex(gp, n, M, code, start, count, _ptr(k1), _ptr(k2_out), walk,
                                  _stream(stream)), "qsim_run_fused_ex")


GRAPH_MAP_GATHER, GRAPH_FUSED, GRAPH_APPLY = 0, 1, 2


class Graph:
    """A CUDA graph of `reps` steps of one planned call (qsim_graph_*)."""

    def __init__(self, plan: Plan, gates, call: int, perm, k1, k2, workspace, reps: int = 1):
        self._g, gp, n = _gates(gates)
        h = ctypes.c_void_p()
        _check(_lib.qsim_graph_create(ctypes.byref(plan), gp, n, call, _ptr(perm), _ptr(k1),
                                      _ptr(k2), _ptr(workspace), reps, ctypes.byref(h)),
               "qsim_graph_create")
        self._h = h
        self._keep = (perm, k1, k2, workspace)   # the graph holds their addresses

    def launch(self, stream=None) -> None:
        _check(_lib.qsim_graph_launch(self._h, _stream(stream)), "qsim_graph_launch")

    def close(self) -> None:
        if self._h:
            _check(_lib.qsim_graph_destroy(self._h), "qsim_graph_destroy")
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_host_batch(gates, M: int, mode: int, k1_hosts, k2_hosts, k1_devs, k2_devs, perm_dev=None,
                   workspace=None, dtype=None) -> None:
    """nsteps = len(k1_hosts) states end to end with overlapped copies (two device
    buffers each for k1 and k2); returns after everything is synchronised."""
    g, gp, n = _gates(gates)
    code = _dtype_code(k1_hosts[0] if dtype is None else dtype)
    ns = len(k1_hosts)
    if len(k2_hosts) != ns or len(k1_devs) != 2 or len(k2_devs) != 2:
        raise ValueError("need nsteps host buffers each and two device buffers each")
    kh1 = (ctypes.c_void_p * max(ns, 1))(*[_ptr(x) for x in k1_hosts])
    kh2 = (ctypes.c_void_p * max(ns, 1))(*[_ptr(x) for x in k2_hosts])
    _check(_lib.qsim_run_host_batch(gp, n, M, code, mode, ns, ctypes.cast(kh1, ctypes.c_void_p),
                                    ctypes.cast(kh2, ctypes.c_void_p), _ptr(k1_devs[0]),
                                    _ptr(k1_devs[1]), _ptr(k2_devs[0]), _ptr(k2_devs[1]),
                                    _ptr(perm_dev), _ptr(workspace)), "qsim_run_host_batch")


def run_host(gates, M: int, mode: int, k1_host, k2_host, k1_dev, k2_dev, perm_dev=None,
             workspace=None, stream=None, dtype=None) -> None:
    """End to end from host buffers; returns after the stream is synchronised."""
    g, gp, n = _gates(gates)
    code = _dtype_code(k1_host if dtype is None else dtype)
    _check(_lib.qsim_run_host(gp, n, M, code, mode, _ptr(k1_host), _ptr(k2_host), _ptr(k1_dev),
                              _ptr(k2_dev), _ptr(perm_dev), _ptr(workspace), _stream(stream)),
           "qsim_run_host")


def plan_create(gates, M: int, dtype="c64") -> Plan:
    g, gp, n = _gates(gates)
    plan = Plan()
    _check(_lib.qsim_plan_create(gp, n, M, _dtype_code(dtype), ctypes.byref(plan)),
           "qsim_plan_create")
    return plan


def plan_tune(plan: Plan, gates, perm, k1, k2, workspace, stream=None, effort=None) -> int:
    """Measure plan variants on these buffers and keep the fastest map + gather
    in `plan` (returns the variant index; see qsim_plan_tune).  effort:
    None / TUNE_PATIENT (all stages, qsim_plan_tune) or TUNE_MEASURE (stages
    1-3, qsim_plan_tune_ex)."""
    g, gp, n = _gates(gates)
    chosen = ctypes.c_int32(-1)
    if effort is None:
        _check(_lib.qsim_plan_tune(ctypes.byref(plan), gp, n, _ptr(perm), _ptr(k1), _ptr(k2),
                                   _ptr(workspace), _stream(stream), ctypes.byref(chosen)),
               "qsim_plan_tune")
    else:
        _check(_lib.qsim_plan_tune_ex(ctypes.byref(plan), gp, n, _ptr(perm), _ptr(k1), _ptr(k2),
                                      _ptr(workspace), _stream(stream), int(effort),
                                      ctypes.byref(chosen)),
               "qsim_plan_tune_ex")
    return chosen.value


def _need_plan(plan: Plan, k1, k2, perm=None, workspace=None) -> None:
    if 1 <= plan.M <= 32 and plan.dtype in _ELEM:
        nb = _ELEM[plan.dtype] << plan.M
        _need(k1, nb, "k1")
        _need(k2, nb, "k2")
        _need(perm, 4 << plan.M, "perm")
        _need(workspace, WORKSPACE_BYTES, "workspace")


def apply_map_planned(plan: Plan, perm, k1, k2, workspace=None, stream=None) -> None:
    """qsim_apply_map in the plan's traversal order (same k2 bytes)."""
    _need_plan(plan, k1, k2, perm, workspace)
    _check(_lib.qsim_apply_map_planned(ctypes.byref(plan), _ptr(perm), _ptr(k1), _ptr(k2),
                                       _ptr(workspace), _stream(stream)),
           "qsim_apply_map_planned")


def run_fused_planned(plan: Plan, gates, k1, k2, workspace=None, stream=None) -> None:
    """qsim_run_fused in the plan's traversal order (same k2 bytes)."""
    g, gp, n = _gates(gates)
    _need_plan(plan, k1, k2, None, workspace)
    _check(_lib.qsim_run_fused_planned(ctypes.byref(plan), gp, n, _ptr(k1), _ptr(k2),
                                       _ptr(workspace), _stream(stream)),
           "qsim_run_fused_planned")


def map_gather_planned(plan: Plan, gates, perm, k1, k2, workspace=None, stream=None) -> None:
    """perm (materialised map) and k2 = k1[perm] in one call (one kernel when JIT)."""
    g, gp, n = _gates(gates)
    _need_plan(plan, k1, k2, perm, workspace)
    _check(_lib.qsim_map_gather_planned(ctypes.byref(plan), gp, n, _ptr(perm), _ptr(k1), _ptr(k2),
                                        _ptr(workspace), _stream(stream)),
           "qsim_map_gather_planned")


def run_fused_kron(gates, M: int, qubits, k2_out, start: int = 0, count: int | None = None,
                   dtype=None, walk: int = WALK_AUTO, stream=None) -> None:
    """k2_out[r] = k1(perm[start + r]) with k1 = q_M (x) ... (x) q_1 generated on
    the fly (Appendix 1).  qubits: (M, 2) complex, row j-1 = [q_j(0), q_j(1)]."""
    q = np.ascontiguousarray(np.asarray(qubits, dtype=np.complex128).reshape(-1, 2))
    if q.shape[0] != M:
        raise ValueError(f"need {M} qubits, got {q.shape[0]}")
    qd = np.ascontiguousarray(q.view(np.float64).reshape(-1))
    if count is None:
        count = (1 << M) - start
    if dtype is None:                    # from the output tensor, else complex64
        dtype = _tensor_dtype(k2_out)
        dtype = C64 if dtype is None else dtype
    code = _dtype_code(dtype)
    td = _tensor_dtype(k2_out)
    if td is not None and td != code:
        raise ValueError(f"k2_out is {k2_out.dtype} but dtype says {dtype}")
    if code in _ELEM:
        _need(k2_out, _ELEM[code] * count, "k2_out")
    g, gp, n = _gates(gates)
    _check(_lib.qsim_run_fused_kron(gp, n, M, code, qd.ctypes.data, start, count,
                                    _ptr(k2_out), walk, _stream(stream)), "qsim_run_fused_kron")


def workspace(device=None):
    """A device workspace of WORKSPACE_BYTES for the planned calls."""
    import torch
    return torch.zeros(WORKSPACE_BYTES, dtype=torch.uint8,
                       device=device if device is not None else "cuda")


def last_kernel() -> str:
    """Kernel the last planned, build_map or run_fused_kron call on this thread
    launched (diagnostics; see qsim_last_kernel in include/qsim.h)."""
    return _lib.qsim_last_kernel().decode()


def jit_status() -> str:
    return _lib.qsim_jit_status().decode()


def jit_last_compile_ms() -> float:
    return float(_lib.qsim_jit_last_compile_ms())


def last_launch_count() -> int:
    return int(_lib.qsim_last_launch_count())
