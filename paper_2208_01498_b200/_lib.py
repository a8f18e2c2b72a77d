"""ctypes marshalling for include/tn.h (same names as the C entry points)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtn_b200.so")

TN_C64, TN_C128 = 0, 1
TN_PATH_AUTO, TN_PATH_SMALL, TN_PATH_TC, TN_PATH_SKINNY, TN_PATH_WIDE = 0, 1, 2, 3, 4

EXPORTED_SYMBOLS = [
    "tn_last_error", "tn_version", "tn_build_network", "tn_network_free", "tn_network_get_info",
    "tn_network_dims", "tn_network_tensor", "tn_order_params_default", "tn_find_order", "tn_order_free",
    "tn_order_get_info", "tn_order_steps", "tn_order_slices", "tn_order_import", "tn_plan_create", "tn_plan_free",
    "tn_plan_get_info", "tn_plan_steps", "tn_plan_set_lanes", "tn_contributing_slices", "tn_contributing_slice_ids", "tn_contract", "tn_contract_device", "tn_contract_profiled", "tn_profile_defer", "tn_profile_collect", "tn_prepare", "tn_contract_prepared", "tn_amplitudes", "tn_contract_pair",
    "tn_kernel_launches",
]


class TnError(RuntimeError):
    pass


class _NetInfo(C.Structure):
    _fields_ = [("n_tensors", C.c_int32), ("n_indices", C.c_int32), ("n_qubits", C.c_int32),
                ("max_rank", C.c_int32), ("radius", C.c_double), ("k_bound", C.c_double)]


class OrderParams(C.Structure):
    _fields_ = [("leaf_size", C.c_int32), ("a_max", C.c_int32), ("n_valid", C.c_int32),
                ("max_tries", C.c_int32), ("n_seeds", C.c_int32), ("max_log2_size", C.c_int32)]


class _OrderInfo(C.Structure):
    _fields_ = [("n_steps", C.c_int32), ("n_slices", C.c_int32), ("max_step_log2", C.c_int32),
                ("max_size_log2", C.c_int32), ("median_fallbacks", C.c_int32),
                ("log2_total_2M", C.c_double), ("log2_slice_2M", C.c_double),
                ("n_slice_assignments", C.c_int64), ("slice_bits", C.c_int32)]


class Profile(C.Structure):
    _fields_ = [("ms_small", C.c_double), ("ms_pack", C.c_double), ("ms_gemm", C.c_double),
                ("ms_other", C.c_double), ("flops_gemm", C.c_double), ("flops_small", C.c_double),
                ("bytes_small", C.c_double), ("bytes_pack", C.c_double), ("n_gemm", C.c_int64),
                ("n_pack", C.c_int64), ("n_small", C.c_int64), ("n_other", C.c_int64),
                ("k_ms", C.c_double * 16), ("k_flops", C.c_double * 16), ("k_bytes", C.c_double * 16),
                ("k_intervals", C.c_int64 * 16)]


# kernel classes of Profile.k_* (include/tn.h TN_K_*)
KERNEL_CLASSES = ["small_contract_kernel", "pack_f16x2s_kernel", "cgemm_f16x2s_kernel", "cgemm2_f16x2s_kernel",
                  "cgemm2p_f16x2s_kernel", "pack_planar_kernel", "zgemm_dmma_kernel", "skinny_kernel",
                  "wide_kernel", "reduce (splitk / skinny)", "other"]


class _PlanInfo(C.Structure):
    _fields_ = [("flops_per_slice", C.c_double), ("n_slices", C.c_int64), ("arena_bytes", C.c_int64),
                ("n_steps_small", C.c_int32), ("n_steps_tc", C.c_int32), ("n_launches_per_slice", C.c_int32),
                ("tc_flops_per_slice", C.c_double), ("slice_bits", C.c_int32), ("flops_prologue", C.c_double),
                ("frontier_bytes", C.c_int64), ("n_launches_prologue", C.c_int32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run paper_2208_01498_b200/build.py (no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    P, I32, I64, D = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    sig = {
        "tn_last_error": (C.c_char_p, []),
        "tn_version": (C.c_char_p, []),
        "tn_build_network": (C.c_int, [I32, P, I32, P, P, I32, C.POINTER(P)]),
        "tn_network_free": (None, [P]),
        "tn_network_get_info": (C.c_int, [P, C.POINTER(_NetInfo)]),
        "tn_network_dims": (C.c_int, [P, P, P]),
        "tn_network_tensor": (C.c_int, [P, I32, P, P, P, P, I64]),
        "tn_order_params_default": (None, [C.POINTER(OrderParams)]),
        "tn_find_order": (C.c_int, [P, C.POINTER(OrderParams), C.c_uint64, C.POINTER(P)]),
        "tn_order_free": (None, [P]),
        "tn_order_import": (C.c_int, [P, P, I32, P, I32, I32, C.POINTER(P)]),
        "tn_order_get_info": (C.c_int, [P, C.POINTER(_OrderInfo)]),
        "tn_order_steps": (C.c_int, [P, P]),
        "tn_order_slices": (C.c_int, [P, P]),
        "tn_plan_create": (C.c_int, [P, P, I32, I32, C.POINTER(P)]),
        "tn_plan_free": (None, [P]),
        "tn_plan_get_info": (C.c_int, [P, C.POINTER(_PlanInfo)]),
        "tn_plan_steps": (C.c_int, [P, P]),
        "tn_plan_set_lanes": (C.c_int, [P, I32]),
        "tn_contributing_slices": (C.c_int, [P, P, C.POINTER(C.c_int64)]),
        "tn_contributing_slice_ids": (C.c_int, [P, P, I64, I64, P, C.POINTER(C.c_int64)]),
        "tn_contract": (C.c_int, [P, P, I64, I64, P, P]),
        "tn_contract_device": (C.c_int, [P, P, I64, I64, P, P]),
        "tn_contract_profiled": (C.c_int, [P, P, I64, I64, P, P, C.POINTER(Profile)]),
        "tn_prepare": (C.c_int, [P, P, P, C.POINTER(Profile)]),
        "tn_profile_defer": (C.c_int, [P, I32]),
        "tn_profile_collect": (C.c_int, [P, C.POINTER(Profile)]),
        "tn_contract_prepared": (C.c_int, [P, I64, I64, P, P, C.POINTER(Profile)]),
        "tn_amplitudes": (C.c_int, [P, P, I32, P, P]),
        "tn_contract_pair": (C.c_int, [I32, P, I32, P, P, I32, P, P, I32, P, P, I32, I32, P]),
        "tn_kernel_launches": (C.c_int64, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L


lib = _load()


def _check(rc):
    if rc != 0:
        raise TnError(f"tn error {rc}: {lib.tn_last_error().decode()}")


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def kernel_launches() -> int:
    return int(lib.tn_kernel_launches())


class Network:
    """tn_build_network: circuit -> closed tensor network."""

    def __init__(self, n_qubits, qubit_xy, gate_qubits, gate_mats, diag_hyper=False):
        xy = np.ascontiguousarray(qubit_xy, dtype=np.float64)
        gq = np.ascontiguousarray(gate_qubits, dtype=np.int32)
        gm = np.ascontiguousarray(np.asarray(gate_mats, dtype=np.complex128).view(np.float64))
        h = C.c_void_p()
        _check(lib.tn_build_network(int(n_qubits), _ptr(xy), int(gq.shape[0]), _ptr(gq), _ptr(gm),
                                    int(bool(diag_hyper)), C.byref(h)))
        self.h = h
        self.n_qubits = int(n_qubits)

    @classmethod
    def from_circuit(cls, circ, diag_hyper=False):
        xy, gq, gm = circ.flat()
        return cls(circ.n, xy, gq, gm, diag_hyper)

    def __del__(self):
        if getattr(self, "h", None):
            lib.tn_network_free(self.h)
            self.h = None

    def info(self):
        i = _NetInfo()
        _check(lib.tn_network_get_info(self.h, C.byref(i)))
        return {k: getattr(i, k) for k, _ in i._fields_}

    def dims(self):
        inf = self.info()
        d = np.zeros(inf["n_indices"], np.int32)
        o = np.zeros(inf["n_qubits"], np.int32)
        _check(lib.tn_network_dims(self.h, _ptr(d), _ptr(o)))
        return d, o

    def tensor(self, t, with_data=True):
        inf = self.info()
        r = C.c_int32()
        inds = np.zeros(max(1, inf["max_rank"]), np.int32)
        pos = np.zeros(2, np.float64)
        _check(lib.tn_network_tensor(self.h, int(t), C.byref(r), _ptr(inds), _ptr(pos), None, 0))
        inds = inds[:r.value].copy()
        data = None
        if with_data:
            d, _ = self.dims()
            n = int(np.prod([d[i] for i in inds])) if len(inds) else 1
            buf = np.zeros(2 * n, np.float64)
            _check(lib.tn_network_tensor(self.h, int(t), C.byref(r), None, None, _ptr(buf), buf.size))
            data = buf.view(np.complex128).reshape([int(d[i]) for i in inds]) if len(inds) else buf.view(np.complex128)[0]
        return inds, pos, data


class Order:
    """tn_find_order: separator hierarchy (SM Algorithm 1) + greedy leaves + slicing."""

    def __init__(self, net: Network, seed=0, max_log2_size=0, **kw):
        p = OrderParams()
        lib.tn_order_params_default(C.byref(p))
        p.max_log2_size = int(max_log2_size)
        for k, v in kw.items():
            setattr(p, k, int(v))
        h = C.c_void_p()
        _check(lib.tn_find_order(net.h, C.byref(p), C.c_uint64(seed), C.byref(h)))
        self.h = h
        self.net = net          # the network must outlive the order

    @classmethod
    def from_steps(cls, net: Network, steps, slices=(), median_fallbacks=0):
        """tn_order_import: an order given as its steps [(a, b), ...] and sliced indices
        (e.g. found by another rank and broadcast, dist.shared_order)."""
        st = np.ascontiguousarray(np.asarray(steps, np.int32).reshape(-1))
        sl = np.ascontiguousarray(np.asarray(list(slices), np.int32))
        st_p = _ptr(st) if st.size else None
        sl_p = _ptr(sl) if sl.size else None
        h = C.c_void_p()
        _check(lib.tn_order_import(net.h, st_p, len(st) // 2, sl_p, len(sl), int(median_fallbacks), C.byref(h)))
        o = cls.__new__(cls)
        o.h = h
        o.net = net
        return o

    def __del__(self):
        if getattr(self, "h", None):
            lib.tn_order_free(self.h)
            self.h = None

    def info(self):
        i = _OrderInfo()
        _check(lib.tn_order_get_info(self.h, C.byref(i)))
        return {k: getattr(i, k) for k, _ in i._fields_}

    def steps(self):
        n = self.info()["n_steps"]
        s = np.zeros(2 * max(n, 1), np.int32)
        _check(lib.tn_order_steps(self.h, _ptr(s)))
        return [(int(s[2 * k]), int(s[2 * k + 1])) for k in range(n)]

    def slices(self):
        n = self.info()["n_slices"]
        s = np.zeros(max(n, 1), np.int32)
        _check(lib.tn_order_slices(self.h, _ptr(s)))
        return [int(v) for v in s[:n]]


class Plan:
    """tn_plan_create / tn_contract / tn_amplitudes on CUDA device `device`."""

    def __init__(self, net: Network, order: Order, dtype=TN_C64, device=0):
        h = C.c_void_p()
        _check(lib.tn_plan_create(net.h, order.h, int(dtype), int(device), C.byref(h)))
        self.h = h
        self.net, self.order, self.dtype = net, order, dtype

    def __del__(self):
        if getattr(self, "h", None):
            lib.tn_plan_free(self.h)
            self.h = None

    def info(self):
        i = _PlanInfo()
        _check(lib.tn_plan_get_info(self.h, C.byref(i)))
        return {k: getattr(i, k) for k, _ in i._fields_}

    def steps(self):
        n = self.order.info()["n_steps"]
        out = np.zeros(6 * max(n, 1), np.int32)
        _check(lib.tn_plan_steps(self.h, _ptr(out)))
        return out[:6 * n].reshape(n, 6)

    def contributing_slices(self, bits):
        """tn_contributing_slices: slices not provably zero for this bitstring."""
        b = np.ascontiguousarray(bits, dtype=np.uint8)
        c = C.c_int64()
        _check(lib.tn_contributing_slices(self.h, _ptr(b), C.byref(c)))
        return int(c.value)

    def contributing_slice_ids(self, bits, slice_begin=0, cap=64):
        """tn_contributing_slice_ids: first `cap` contributing slice ids >= slice_begin."""
        b = np.ascontiguousarray(bits, dtype=np.uint8)
        out = np.zeros(max(int(cap), 1), np.int64)
        c = C.c_int64()
        _check(lib.tn_contributing_slice_ids(self.h, _ptr(b), int(slice_begin), int(cap), _ptr(out), C.byref(c)))
        return [int(v) for v in out[:c.value]]

    def set_lanes(self, n_lanes):
        """tn_plan_set_lanes: n_lanes concurrent copies of the per-contraction state."""
        _check(lib.tn_plan_set_lanes(self.h, int(n_lanes)))

    def contract(self, bits, slice_begin=0, slice_end=None, stream=None):
        b = np.ascontiguousarray(bits, dtype=np.uint8)
        if slice_end is None:
            slice_end = self.info()["n_slices"]
        out = np.zeros(2, np.float64)
        _check(lib.tn_contract(self.h, _ptr(b), int(slice_begin), int(slice_end), _ptr(out),
                               C.c_void_p(stream or 0)))
        return complex(out[0], out[1])

    def contract_device(self, bits_dev_ptr, slice_begin, slice_end, amp_dev_ptr, stream=0):
        _check(lib.tn_contract_device(self.h, C.c_void_p(bits_dev_ptr), int(slice_begin), int(slice_end),
                                      C.c_void_p(amp_dev_ptr), C.c_void_p(stream)))

    def contract_profiled(self, bits_dev_ptr, slice_begin, slice_end, amp_dev_ptr, stream=0):
        pr = Profile()
        _check(lib.tn_contract_profiled(self.h, C.c_void_p(bits_dev_ptr), int(slice_begin), int(slice_end),
                                        C.c_void_p(amp_dev_ptr), C.c_void_p(stream), C.byref(pr)))
        return self._profile_dict(pr)

    @staticmethod
    def _profile_dict(pr):
        out = {k: getattr(pr, k) for k, _ in pr._fields_ if not k.startswith("k_")}
        out["kernels"] = {name: {"ms": pr.k_ms[i], "flops": pr.k_flops[i], "bytes": pr.k_bytes[i],
                                 "intervals": int(pr.k_intervals[i])}
                          for i, name in enumerate(KERNEL_CLASSES)}
        return out

    def profile_defer(self, on=True):
        """tn_profile_defer: profiled calls stop waiting for their kernels; their device
        times are collected by profile_collect()."""
        _check(lib.tn_profile_defer(self.h, 1 if on else 0))

    def profile_collect(self):
        """tn_profile_collect: waits for the deferred profiled replays, returns their summed
        device times (profile dict, flops / bytes zero)."""
        pr = Profile()
        _check(lib.tn_profile_collect(self.h, C.byref(pr)))
        return self._profile_dict(pr)

    def prepare(self, bits_dev_ptr, stream=0, profiled=False):
        """tn_prepare: the bitstring's slice-invariant prologue (profile dict if profiled)."""
        pr = Profile() if profiled else None
        _check(lib.tn_prepare(self.h, C.c_void_p(bits_dev_ptr), C.c_void_p(stream), C.byref(pr) if profiled else None))
        return self._profile_dict(pr) if profiled else None

    def contract_prepared(self, slice_begin, slice_end, amp_dev_ptr, stream=0, profiled=False):
        """tn_contract_prepared: slices of the prepared bitstring (profile dict if profiled)."""
        pr = Profile() if profiled else None
        _check(lib.tn_contract_prepared(self.h, int(slice_begin), int(slice_end), C.c_void_p(amp_dev_ptr),
                                        C.c_void_p(stream), C.byref(pr) if profiled else None))
        return self._profile_dict(pr) if profiled else None

    def amplitudes(self, bits, stream=None):
        b = np.ascontiguousarray(bits, dtype=np.uint8)
        n = b.shape[0]
        out = np.zeros(2 * n, np.float64)
        _check(lib.tn_amplitudes(self.h, _ptr(b), int(n), _ptr(out), C.c_void_p(stream or 0)))
        return out.view(np.complex128)


def contract_pair(dtype, A_ptr, inds_a, B_ptr, inds_b, C_ptr, inds_c, dims, path=TN_PATH_AUTO, stream=0):
    """tn_contract_pair on device buffers (pointers as ints)."""
    ia = np.ascontiguousarray(inds_a, np.int32)
    ib = np.ascontiguousarray(inds_b, np.int32)
    ic = np.ascontiguousarray(inds_c, np.int32)
    d = np.ascontiguousarray(dims, np.int32)
    _check(lib.tn_contract_pair(int(dtype), C.c_void_p(A_ptr), len(ia), _ptr(ia), C.c_void_p(B_ptr), len(ib),
                                _ptr(ib), C.c_void_p(C_ptr), len(ic), _ptr(ic), _ptr(d), len(d), int(path),
                                C.c_void_p(stream)))
