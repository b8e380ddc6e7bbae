"""TEST INFRASTRUCTURE ONLY -- ctypes loaders for the CPU checkers.

* ``Oracle``    : oracle/_build/libtfla_oracle.so, the plain-C f64 restatement
                  of the reference chunkwise path (oracle/tfla_oracle.c).
* ``Reference`` : oracle/_ref/libmlstm_ref.so, the unmodified reference C++
                  library compiled from /root/reference/proj/src with a C shim
                  (oracle/ref_shim.cpp). Absent when it was never built.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and the
``--impl reference`` arm) may import this module; the product path never does.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "_build" / "libtfla_oracle.so"
REF_SO = HERE / "_ref" / "libmlstm_ref.so"

_D = ctypes.POINTER(ctypes.c_double)
_L = ctypes.c_long


def _p(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_D)


def _zeros(*shape):
    return np.zeros(shape, dtype=np.float64)


class _Base:
    def fwd_shapes(self, B, H, T, L, dqk, dhv):
        NC = T // L
        return dict(
            h=(B, H, T, dhv),
            C=(B, H, NC + 1, dqk, dhv),
            n=(B, H, NC + 1, dqk),
            m=(B, H, NC + 1),
            m_comb=(B, H, T),
            h_denom=(B, H, T),
        )


class Oracle(_Base):
    """The C restatement (f64)."""

    def __init__(self, path: Path | None = None):
        path = Path(path or ORACLE_SO)
        if not path.exists():
            raise RuntimeError(f"oracle not built: {path} (make oracle)")
        self.lib = ctypes.CDLL(str(path))
        self.threads = int(os.environ.get("TFLA_ORACLE_THREADS", os.cpu_count() or 1))

    def gates(self, f_pre, i_pre, L, variant):
        T = f_pre.shape[0]
        g, b, a = _zeros(T // L), _zeros(T), _zeros(T)
        rc = self.lib.or_chunkwise_gates(_p(f_pre), _p(i_pre), _L(T), _L(L), variant, _p(g), _p(b), _p(a))
        assert rc == 0
        return g, b, a

    def forward(self, q, k, v, i_pre, f_pre, L, variant):
        B, H, T, dqk = q.shape
        dhv = v.shape[-1]
        out = {n: _zeros(*s) for n, s in self.fwd_shapes(B, H, T, L, dqk, dhv).items()}
        rc = self.lib.or_forward(
            _L(B), _L(H), _L(T), _L(L), _L(dqk), _L(dhv), variant,
            _p(q), _p(k), _p(v), _p(i_pre), _p(f_pre),
            _p(out["h"]), _p(out["C"]), _p(out["n"]), _p(out["m"]), _p(out["m_comb"]), _p(out["h_denom"]),
            self.threads,
        )
        assert rc == 0
        return out

    def backward(self, q, k, v, i_pre, f_pre, dh, C, m, m_comb, h_denom, L, variant):
        B, H, T, dqk = q.shape
        dhv = v.shape[-1]
        g = dict(dq=_zeros(B, H, T, dqk), dk=_zeros(B, H, T, dqk), dv=_zeros(B, H, T, dhv),
                 d_fpre=_zeros(B, H, T), d_ipre=_zeros(B, H, T))
        rc = self.lib.or_backward(
            _L(B), _L(H), _L(T), _L(L), _L(dqk), _L(dhv), variant,
            _p(q), _p(k), _p(v), _p(i_pre), _p(f_pre), _p(dh), _p(C), _p(m), _p(m_comb), _p(h_denom),
            _p(g["dq"]), _p(g["dk"]), _p(g["dv"]), _p(g["d_fpre"]), _p(g["d_ipre"]),
            self.threads,
        )
        assert rc == 0
        return g

    def backward_parts(self, q, k, v, i_pre, f_pre, dh, C, m, m_comb, h_denom, L, variant):
        """backward plus the split-entry-point partials: d_b_q (TfLaDqResult::d_b_cum),
        d_b_kv / d_a_tail / d_i_log (TfLaDkResult), d_g / d_c (backward_state_pass_head)."""
        B, H, T, dqk = q.shape
        dhv = v.shape[-1]
        NC = T // L
        g = dict(dq=_zeros(B, H, T, dqk), dk=_zeros(B, H, T, dqk), dv=_zeros(B, H, T, dhv),
                 d_fpre=_zeros(B, H, T), d_ipre=_zeros(B, H, T), d_b_q=_zeros(B, H, T),
                 d_b_kv=_zeros(B, H, T), d_a_tail=_zeros(B, H, T), d_i_log=_zeros(B, H, T),
                 d_g=_zeros(B, H, NC), d_c=_zeros(B, H, NC + 1, dqk, dhv))
        rc = self.lib.or_backward_parts(
            _L(B), _L(H), _L(T), _L(L), _L(dqk), _L(dhv), variant,
            _p(q), _p(k), _p(v), _p(i_pre), _p(f_pre), _p(dh), _p(C), _p(m), _p(m_comb), _p(h_denom),
            _p(g["dq"]), _p(g["dk"]), _p(g["dv"]), _p(g["d_fpre"]), _p(g["d_ipre"]),
            _p(g["d_b_q"]), _p(g["d_b_kv"]), _p(g["d_a_tail"]), _p(g["d_i_log"]), _p(g["d_g"]), _p(g["d_c"]),
            self.threads,
        )
        assert rc == 0
        return g

    def recurrent(self, q, k, v, i_pre, f_pre, variant, C_init=None, n_init=None, m_init=None):
        """run_recurrent (recurrent.cpp:65-115) with an optional initial state."""
        B, H, T, dqk = q.shape
        dhv = v.shape[-1]
        out = dict(h=_zeros(B, H, T, dhv), C=_zeros(B, H, dqk, dhv), n=_zeros(B, H, dqk), m=_zeros(B, H))
        rc = self.lib.or_recurrent(
            _L(B), _L(H), _L(T), _L(dqk), _L(dhv), variant, _p(q), _p(k), _p(v), _p(i_pre), _p(f_pre),
            _p(C_init), _p(n_init), _p(m_init), _p(out["h"]), _p(out["C"]), _p(out["n"]), _p(out["m"]))
        assert rc == 0
        return out


    def output_norm_gate(self, h_tilde, o_pre, gamma, eps):
        """h = sigmoid(o_pre) * rms_norm(h_tilde; gamma[h], eps) (eq. 5, transfer.cpp:8-18)."""
        B, H, T, dhv = h_tilde.shape
        out = _zeros(B, H, T, dhv)
        rc = self.lib.or_output_norm_gate(_L(B), _L(H), _L(T), _L(dhv), _p(h_tilde), _p(o_pre), _p(gamma),
                                          ctypes.c_double(eps), _p(out))
        assert rc == 0
        return out


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Reference(_Base):
    """The reference library itself (f64), via oracle/ref_shim.cpp."""

    def __init__(self, path: Path | None = None):
        path = Path(path or REF_SO)
        if not path.exists():
            raise RuntimeError(f"reference not built: {path} (make oracle in the build container)")
        self.lib = ctypes.CDLL(str(path))
        self.lib.ref_last_error.restype = ctypes.c_char_p
        self.lib.ref_stab_checks.restype = ctypes.c_longlong
        self.lib.ref_stab_violations.restype = ctypes.c_longlong

    @staticmethod
    def available() -> bool:
        return REF_SO.exists()

    def _check(self, rc):
        if rc != 0:
            raise RefError(rc, self.lib.ref_last_error().decode())

    def make_inputs(self, B, H, T, dqk, dhv, seed, scale=1.0, gate_scale=1.0):
        q, k = _zeros(B, H, T, dqk), _zeros(B, H, T, dqk)
        v = _zeros(B, H, T, dhv)
        ip, fp = _zeros(B, H, T), _zeros(B, H, T)
        self._check(self.lib.ref_make_inputs(
            _L(B), _L(H), _L(T), _L(dqk), _L(dhv), ctypes.c_uint64(seed), ctypes.c_double(scale),
            ctypes.c_double(gate_scale), _p(q), _p(k), _p(v), _p(ip), _p(fp)))
        return q, k, v, ip, fp

    def normals(self, seed, skip, n, scale=1.0):
        out = _zeros(n)
        self._check(self.lib.ref_normals(ctypes.c_uint64(seed), _L(skip), _L(n), ctypes.c_double(scale), _p(out)))
        return out

    def gates(self, f_pre, i_pre, L, variant):
        T = f_pre.shape[0]
        g, b, a = _zeros(T // L), _zeros(T), _zeros(T)
        self._check(self.lib.ref_chunkwise_gates(_p(f_pre), _p(i_pre), _L(T), _L(L), variant, _p(g), _p(b), _p(a)))
        return g, b, a

    @staticmethod
    def _blocks(blocks):
        if blocks is None:
            return None
        arr = (ctypes.c_long * 4)(*blocks)
        return arr

    def forward(self, q, k, v, i_pre, f_pre, L, variant, blocks=None):
        B, H, T, dqk = q.shape
        dhv = v.shape[-1]
        out = {n: _zeros(*s) for n, s in self.fwd_shapes(B, H, T, L, dqk, dhv).items()}
        self._check(self.lib.ref_forward(
            _L(B), _L(H), _L(T), _L(L), _L(dqk), _L(dhv), variant, self._blocks(blocks),
            _p(q), _p(k), _p(v), _p(i_pre), _p(f_pre),
            _p(out["h"]), _p(out["C"]), _p(out["n"]), _p(out["m"]), _p(out["m_comb"]), _p(out["h_denom"])))
        return out

    def backward(self, q, k, v, i_pre, f_pre, dh, C, n, m, m_comb, h_denom, L, variant, blocks=None):
        B, H, T, dqk = q.shape
        dhv = v.shape[-1]
        g = dict(dq=_zeros(B, H, T, dqk), dk=_zeros(B, H, T, dqk), dv=_zeros(B, H, T, dhv),
                 d_fpre=_zeros(B, H, T), d_ipre=_zeros(B, H, T))
        self._check(self.lib.ref_backward(
            _L(B), _L(H), _L(T), _L(L), _L(dqk), _L(dhv), variant, self._blocks(blocks),
            _p(q), _p(k), _p(v), _p(i_pre), _p(f_pre), _p(dh), _p(C), _p(n), _p(m), _p(m_comb), _p(h_denom),
            _p(g["dq"]), _p(g["dk"]), _p(g["dv"]), _p(g["d_fpre"]), _p(g["d_ipre"])))
        return g

    def backward_split(self, q, k, v, i_pre, f_pre, dh, C, n, m, m_comb, h_denom, L, variant, blocks):
        """tfla_backward_dq / _dk / _dv + backward_state_pass_head of the reference."""
        B, H, T, dqk = q.shape
        dhv = v.shape[-1]
        NC = T // L
        g = dict(dq=_zeros(B, H, T, dqk), d_b_q=_zeros(B, H, T), dk=_zeros(B, H, T, dqk),
                 d_a_tail=_zeros(B, H, T), d_b_kv=_zeros(B, H, T), d_i_log=_zeros(B, H, T),
                 dv=_zeros(B, H, T, dhv), d_g=_zeros(B, H, NC), d_c=_zeros(B, H, NC + 1, dqk, dhv))
        self._check(self.lib.ref_backward_split(
            _L(B), _L(H), _L(T), _L(L), _L(dqk), _L(dhv), variant, self._blocks(blocks),
            _p(q), _p(k), _p(v), _p(i_pre), _p(f_pre), _p(dh), _p(C), _p(n), _p(m), _p(m_comb), _p(h_denom),
            *[_p(g[x]) for x in ("dq", "d_b_q", "dk", "d_a_tail", "d_b_kv", "d_i_log", "dv", "d_g", "d_c")]))
        return g

    def has_perfmodel(self) -> bool:
        return hasattr(self.lib, "ref_perfmodel_eval")

    def perfmodel(self, variant, B, H, T, L, dqk, dhv, params, flops_per_s, bytes_per_s):
        """The reference cost model (perfmodel.cpp) at one point: 42 values
        (flops_chunkwise exact / simplified items, flops_parallel, flops_recurrent,
        memops x3, closed forms, optimal L, runtimes, intensities, argmins)."""
        out = _zeros(42)
        prm = np.ascontiguousarray(params, dtype=np.float64)
        self._check(self.lib.ref_perfmodel_eval(
            variant, _L(B), _L(H), _L(T), _L(L), _L(dqk), _L(dhv), _p(prm), ctypes.c_double(flops_per_s),
            ctypes.c_double(bytes_per_s), _p(out)))
        return out

    def recurrent(self, q, k, v, i_pre, f_pre, variant):
        B, H, T, dqk = q.shape
        dhv = v.shape[-1]
        h, C, n, m = _zeros(B, H, T, dhv), _zeros(B, H, dqk, dhv), _zeros(B, H, dqk), _zeros(B, H)
        self._check(self.lib.ref_run_recurrent(
            _L(B), _L(H), _L(T), _L(dqk), _L(dhv), variant, _p(q), _p(k), _p(v), _p(i_pre), _p(f_pre),
            _p(h), _p(C), _p(n), _p(m)))
        return dict(h=h, C_final=C, n_final=n, m_final=m)

    def rms_norm(self, x, gamma, eps):
        """rms_norm (transfer.cpp:8-18) over the last axis."""
        d = x.shape[-1]
        y = np.zeros_like(x)
        self._check(self.lib.ref_rms_norm(_L(x.size // d), _L(d), _p(x), _p(gamma), ctypes.c_double(eps), _p(y)))
        return y

    def parallel(self, q, k, v, i_pre, f_pre, variant):
        B, H, T, dqk = q.shape
        h = _zeros(B, H, T, v.shape[-1])
        self._check(self.lib.ref_parallel_forward(
            _L(B), _L(H), _L(T), _L(dqk), _L(v.shape[-1]), variant, _p(q), _p(k), _p(v), _p(i_pre), _p(f_pre), _p(h)))
        return h

    def gradcheck(self, q, k, v, i_pre, f_pre, w, L, variant, blocks=None, step=1e-6):
        _, _, T, dqk = q.shape
        rep = _zeros(5)
        self._check(self.lib.ref_gradcheck(
            _L(T), _L(L), _L(dqk), _L(v.shape[-1]), variant, self._blocks(blocks),
            _p(q), _p(k), _p(v), _p(i_pre), _p(f_pre), _p(w), ctypes.c_double(step), _p(rep)))
        return dict(zip(("dq", "dk", "dv", "d_fpre", "d_ipre"), rep))

    def time_slices(self, T, L, dqk, dhv, variant, n_slices, threads, tiled=False, with_backward=True, seed=1000):
        f, tot = ctypes.c_double(), ctypes.c_double()
        self._check(self.lib.ref_time_slices(
            _L(T), _L(L), _L(dqk), _L(dhv), variant, int(tiled), _L(n_slices), int(threads),
            int(with_backward), ctypes.c_uint64(seed), ctypes.byref(f), ctypes.byref(tot)))
        return f.value, tot.value


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round f64 values to the nearest bf16 (round-to-nearest-even), back to f64."""
    f = x.astype(np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def max_rel(a: np.ndarray, ref: np.ndarray) -> float:
    """gradcheck.cpp:7-10 convention: max|a - ref| / max(max|ref|, 1e-12)."""
    scale = max(float(np.abs(ref).max()) if ref.size else 0.0, 1e-12)
    return float(np.abs(a - ref).max()) / scale if ref.size else 0.0
