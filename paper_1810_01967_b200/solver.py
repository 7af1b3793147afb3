"""Inexact iterative projected gradient (IPG) with step-size shrinkage, on the GPU.

Drop-in for the reference ``coverblip.solver`` on the exact-projection path:
``SolverConfig`` (``solver.py:43-66``), ``SolveTrace`` (``:69-93``),
``ParameterMaps`` (``:96-101``), ``SolverError`` (``:39-40``), ``step_shrinkage``
(``:116-144``), ``solve`` / ``solve_compressed`` (``:260-275``) and the loop of
``_solve_core`` (``:155-257``).

Device-resident loop (complex64 state, fp64 reductions): per iteration one fused
adjoint+compress for the gradient, r fused projection trials
(``cbb_project_step``: Z = X - mu G, tcgen05 matched filter, fp64 rescoring,
write-back, dX and ||dX||^2) each followed by ||A dX||^2 (decompress + FFT +
gather + norm, nothing stored), and one apply for the new fidelity whose residual
is reused as the next gradient's input (the reference re-applies A for the same
X).  Host work per trial is two 8-byte reads for the accept test
``mu <= ||dX||^2 / ||A dX||^2`` (non-strict, ``solver.py:137``).

``mode="coverblip"`` runs the same exact projection (the cover-tree search is the
CPU baseline this path replaces; with epsilon = 0 the reference's coverblip is
bitwise the exact path, ``test_solver.py:67-84``); it still requires a tree
argument like the reference (``solver.py:167-168``).
"""

from __future__ import annotations

import csv
import ctypes
import math
import threading
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .device import workspace
from .dictionary import atoms_of, device_dictionary, lookup_table_of
from .forward_model import as_device_operator
from .projection import project_cone_exact  # noqa: F401  (re-exported drop-in)

__all__ = ["SolverConfig", "SolveTrace", "ParameterMaps", "SolverError", "step_shrinkage",
           "solve", "solve_compressed", "IpgState"]

_MODES = ("tm", "blip_exact", "coverblip")


class SolverError(RuntimeError):
    pass


@dataclass
class SolverConfig:
    mode: str = "coverblip"
    epsilon: float = 0.0
    mu_init: float | None = None
    zeta: float = 2.0
    max_iters: int = 50
    rel_tol: float = 1e-6
    max_shrink_per_iter: int = 60
    compressed: int | None = None
    step_policy: str = "reset_each_iter"
    fixed_step: float | None = None
    weights_enabled: bool = False
    seed: int = 0

    def __post_init__(self):
        if self.mode not in _MODES:
            raise ValueError(f"unknown mode {self.mode!r}")
        if self.epsilon < 0:
            raise ValueError("epsilon must be nonnegative")
        if self.zeta <= 1:
            raise ValueError("zeta must exceed 1")
        if self.step_policy not in ("reset_each_iter", "carry_over"):
            raise ValueError(f"unknown step policy {self.step_policy!r}")


@dataclass
class SolveTrace:
    records: list = field(default_factory=list)
    iterations: int = 0
    total_cost: int = 0
    total_time: float = 0.0

    def add(self, **rec):
        self.records.append(rec)
        self.iterations = len(self.records)
        self.total_cost += rec.get("cost", 0)

    def fidelities(self):
        return [r["fidelity"] for r in self.records]

    def to_csv(self, path):
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["iter", "fidelity", "mu", "shrinks", "cost", "nmse", "seconds"])
            for r in self.records:
                w.writerow([r["iter"], repr(r["fidelity"]), repr(r["mu"]), r["shrinks"],
                            r["cost"], "" if r["nmse"] is None else repr(r["nmse"]),
                            repr(r["seconds"])])


@dataclass
class ParameterMaps:
    t1: np.ndarray
    t2: np.ndarray
    b0: np.ndarray
    pd: np.ndarray


def step_shrinkage(X, G, mu0, project_fn, apply_diff, zeta, max_shrink, fixed=False):
    """solver.py:116-144 (generic host form, works with any projection / operator callables)."""
    mu = mu0
    shrinks = 0
    while True:
        proj = project_fn(X - mu * G)
        dX = proj.projected - X
        nd = float(np.linalg.norm(dX) ** 2)
        if nd == 0.0:
            return mu, proj, shrinks, True
        if fixed:
            return mu, proj, shrinks, False
        den = float(np.linalg.norm(apply_diff(dX)) ** 2)
        ratio = np.inf if den == 0.0 else nd / den
        if mu <= ratio:
            return mu, proj, shrinks, False
        mu /= zeta
        shrinks += 1
        if shrinks > max_shrink:
            raise SolverError(
                "step-size collapse: shrinkage exceeded "
                f"{max_shrink} sub-iterations")


def _maps_from(dictionary, indices, gammas) -> ParameterMaps:
    """solver.py:147-152."""
    table = lookup_table_of(dictionary)
    if table is None:
        nan = np.full(len(indices), np.nan)
        return ParameterMaps(t1=nan, t2=nan.copy(), b0=nan.copy(), pd=gammas.copy())
    rows = np.asarray(table)[indices]
    return ParameterMaps(t1=rows[:, 0].copy(), t2=rows[:, 1].copy(), b0=rows[:, 2].copy(),
                         pd=gammas.copy())


class IpgState:
    """Device-resident IPG state and the fused kernels of one solve (one GPU)."""

    def __init__(self, Y, A, dictionary, basis, weights, device):
        lib = _lib.load()
        self.lib = lib
        self.A = A
        self.dev = device
        self.dd = device_dictionary(dictionary, device)
        self.n, self.m, self.L = A.n, A.m, A.L
        self.cm = getattr(A, "c", 1) * A.m                            # measurement columns
        self.dim = self.dd.s
        self.V = (None if basis is None else
                  torch.from_numpy(np.ascontiguousarray(basis, dtype=np.complex64)).to(device))
        self.Y = torch.empty((self.L, self.cm), dtype=torch.complex64, device=device)
        self.w = None
        self.load_measurements(Y, weights)
        c64 = dict(dtype=torch.complex64, device=device)
        n, dim = self.n, self.dim
        self.X = torch.zeros((n, dim), **c64)
        self.Xn = torch.empty((n, dim), **c64)
        self.G = torch.empty((n, dim), **c64)
        self.Z = torch.empty((n, dim), **c64)
        self.dX = torch.empty((n, dim), **c64)
        self.AX = torch.zeros((self.L, self.cm), **c64)
        self.R = torch.empty((self.L, self.cm), **c64)
        self.idx = torch.zeros(n, dtype=torch.int32, device=device)
        self.idx_n = torch.zeros(n, dtype=torch.int32, device=device)
        self.gam = torch.zeros(n, dtype=torch.float64, device=device)
        self.gam_n = torch.empty(n, dtype=torch.float64, device=device)
        self.scal = torch.zeros(8, dtype=torch.float64, device=device)  # device scalars
        self.host = torch.zeros(8, dtype=torch.float64, pin_memory=True)
        # sized for the dictionary: includes the split screen's tile-pruning buffers
        self.pws_bytes = lib.cbb_project_workspace_bytes_dict(n, ctypes.byref(self.dd.view))
        self.rws_bytes = lib.cbb_reduce_workspace_bytes()
        self.algo = 0
        self._graphs = {}          # device-decided iteration graphs, per buffer parity

    def _rws(self):
        """The state's own reduction workspace (allocated once: the captured iteration graphs
        point at it, and one solve drives a state at a time)."""
        buf = self.__dict__.get("_rws_buf")
        if buf is None:
            buf = self._rws_buf = torch.empty(max(int(self.rws_bytes), 256), dtype=torch.uint8,
                                              device=self.dev)
        return buf

    def project_workspace(self):
        """The state's own projection workspace (sized for the dictionary's tile pruning)."""
        buf = self.__dict__.get("_pws_buf")
        if buf is None:
            buf = self._pws_buf = torch.empty(max(int(self.pws_bytes), 256), dtype=torch.uint8,
                                              device=self.dev)
        return buf

    def load_measurements(self, Y, weights):
        """Upload Y in the caller's layout and precision into the frame-major complex64 buffer
        (||Y|| in fp64 and the transpose / cast happen on the device) and the loss weights."""
        Yh = np.asarray(Y)
        if Yh.shape != (self.cm, self.L):
            raise ValueError(f"measurements are {Yh.shape}, the operator expects "
                             f"{(self.cm, self.L)}")
        if not np.iscomplexobj(Yh):
            Yh = Yh.astype(np.complex128)
        Yd = torch.from_numpy(np.ascontiguousarray(Yh)).to(self.dev)     # (c*m, L)
        self.y_norm = float(torch.linalg.vector_norm(torch.view_as_real(Yd), dtype=torch.float64))
        self.Y.copy_(Yd.transpose(0, 1))                                  # (L, c*m) complex64
        del Yd
        w = (None if weights is None else torch.from_numpy(np.ascontiguousarray(
            np.broadcast_to(weights, Yh.shape).T, dtype=np.float32)).to(self.dev))
        if w is None or self.w is None:
            self.w = w
        else:
            self.w.copy_(w)                   # keep the buffer a captured graph points to

    def reset_iterates(self):
        """X = 0 (solver.py:199): the state a solve starts from."""
        self.X.zero_()
        self.AX.zero_()
        self.idx.zero_()
        self.gam.zero_()
        self.scal.zero_()

    def read(self, *slots):
        """Device fp64 scalars -> host floats (one small synchronous copy)."""
        k = max(slots) + 1
        self.host[:k].copy_(self.scal[:k], non_blocking=True)
        stream = self.__dict__.get("stream")
        if stream is None:  # the solve's stream, looked up once (the lookup costs ~10 us)
            stream = self.stream = torch.cuda.current_stream(self.dev)
        stream.synchronize()
        return [float(self.host[i]) for i in slots]

    # -- operator chain in the solver's coordinates (compressed or not)
    def apply(self, Xs, out):
        if self.V is not None:
            self.A.fm_apply_compressed(Xs, self.V, out=out)
        else:
            out.copy_(self.A.fm_apply(Xs))
        return out

    def apply_norm2(self, Xs, slot):
        o = self.scal[slot:slot + 1]
        if self.V is not None:
            self.A.fm_apply_norm2_compressed(Xs, self.V, o)
        else:
            Y = self.A.fm_apply(Xs)
            _lib.check(self.lib.cbb_norm2_c64(Y.data_ptr(), Y.numel(), o.data_ptr(),
                                              self._rws().data_ptr(), _lib.stream_ptr()),
                       "norm2")

    def cold_hint(self):
        """Warm-start atoms for an iterate without any (X = 0, the first iteration): the
        argmax over the dictionary's tile representatives of Z = -mu G (mu > 0 does not change
        the argmax), mapped to atom indices, in place of the all-zero idx.  Only a hint: the
        projection's result does not depend on it."""
        reps = self.dd.representatives()
        if reps is None:
            return
        from .projection import project_device
        atoms_idx, rdd = reps
        ridx, _, _ = project_device(-self.G, rdd, idx_int64=True, proj_c128=False)
        self.idx.copy_(atoms_idx[ridx])

    rep_hint_min_voxels = 1 << 18  # measured: pays at cfg4 (4.2 M voxels), neutral at cfg2 (65,536)

    def rep_hint_ready(self) -> bool:
        """Prepare (outside any graph capture) the representatives of a prune-capable dictionary;
        True if first trials get the representative hint (large pruned projections only)."""
        ok = self.__dict__.get("_rep_ok")
        if ok is None:
            ok = self._rep_ok = (self.n >= self.rep_hint_min_voxels
                                 and self.dd.representatives() is not None)
        return ok

    def rep_hint(self, mu, mu_dev=None):
        """First trial of an iteration (k >= 2): idx_n -- which only repeats older atoms there --
        becomes the best tile representative of Z = X - mu G (cbb_project_hint).  After a large
        step the current atoms bound the maximum poorly and the pruned lists grow 2-3x (cfg4:
        0.2-0.6 of all tiles listed without it, 0.15-0.2 with it)."""
        atoms_idx, rdd = self.dd.representatives()
        ws = self.project_workspace()
        _lib.check(self.lib.cbb_project_hint(
            self.X.data_ptr(), self.G.data_ptr(), float(mu), mu_dev, self.Z.data_ptr(), self.n,
            ctypes.byref(rdd.view), atoms_idx.data_ptr(), self.idx_n.data_ptr(), ws.data_ptr(),
            self.pws_bytes, _lib.stream_ptr()), "cbb_project_hint")

    def gradient(self):
        """G = compress(A^H R) with R = w (A X - Y) from the last fidelity evaluation."""
        if self.V is not None:
            self.A.fm_adjoint_compressed(self.R, self.V, out=self.G)
        else:
            self.G.copy_(self.A.fm_adjoint(self.R))

    def residual(self, slot):
        """R = w (AX - Y), scal[slot] = sum w |AX - Y|^2 (solver.py:180-190)."""
        o = self.scal[slot:slot + 1]
        _lib.check(self.lib.cbb_residual(self.AX.data_ptr(), self.Y.data_ptr(), self.AX.numel(),
                                         None if self.w is None else self.w.data_ptr(),
                                         self.R.data_ptr(), o.data_ptr(), self._rws().data_ptr(),
                                         _lib.stream_ptr()), "residual")

    def scaled_obj(self, alpha, slot):
        o = self.scal[slot:slot + 1]
        _lib.check(self.lib.cbb_scaled_residual_norm2(
            self.AX.data_ptr(), float(alpha), self.Y.data_ptr(), self.AX.numel(),
            None if self.w is None else self.w.data_ptr(), o.data_ptr(), self._rws().data_ptr(),
            _lib.stream_ptr()), "scaled_residual")

    def norm2(self, t, slot):
        o = self.scal[slot:slot + 1]
        _lib.check(self.lib.cbb_norm2_c64(t.data_ptr(), t.numel(), o.data_ptr(),
                                          self._rws().data_ptr(), _lib.stream_ptr()), "norm2")

    def scale(self, t, alpha):
        _lib.check(self.lib.cbb_scale_c64(t.data_ptr(), float(alpha), t.numel(),
                                          _lib.stream_ptr()), "scale")

    def project_step(self, mu, slot, mu_dev=None):
        """Xn = P(X - mu G), dX = Xn - X, scal[slot] = ||dX||^2 (solver.py:128-130).  Warm
        start: the current atoms (idx) and the previous trial's winners (idx_n, still in place
        until this projection overwrites them) -- any atom's exact score bounds the maximum."""
        ws = self.project_workspace()
        o = self.scal[slot:slot + 1]
        _lib.check(self.lib.cbb_project_step_ex(
            self.X.data_ptr(), self.G.data_ptr(), float(mu), mu_dev, self.Z.data_ptr(), self.n,
            ctypes.byref(self.dd.view), self.idx.data_ptr(), self.idx_n.data_ptr(),
            self.idx_n.data_ptr(), self.gam_n.data_ptr(), self.Xn.data_ptr(), self.dX.data_ptr(),
            o.data_ptr(), ws.data_ptr(), self.pws_bytes, self.algo, _lib.stream_ptr()),
            "cbb_project_step_ex")

    def decompress(self, Xs):
        return Xs if self.V is None else Xs @ self.V.conj().transpose(0, 1)

    # -- device-decided iterations: one CUDA graph per iteration (include/coverblip_b200.h
    #    cbb_graph_*): gradient, a while-conditional node repeating the trial until the device
    #    accepts mu (solver.py:116-144), the apply of the new iterate and the residual; the host
    #    synchronises once per iteration instead of once per trial.
    _TS_DTYPE = np.dtype([("mu", "<f8"), ("mu_base", "<f8"), ("mu32", "<f4"), ("shrinks", "<i4"),
                          ("fixed", "<i4"), ("status", "<i4"), ("trials", "<i4")])

    def graph_capable(self, config) -> bool:
        """The captured iteration needs allocation-free calls: the s-channel Cartesian
        operator, the adaptive step rule and one GPU (the sharded state all-reduces on read)."""
        return (self.V is not None and getattr(self.A, "kind", "") == "cartesian_dft"
                and int(self.V.shape[1]) <= 32 and config.fixed_step is None
                and type(self) is IpgState)

    def _graph_setup(self):
        if "ts" in self.__dict__:
            return
        nb = int(self.lib.cbb_trial_state_bytes())
        assert nb >= self._TS_DTYPE.itemsize
        self.ts = torch.zeros(nb, dtype=torch.uint8, device=self.dev)
        self.ts_host = torch.zeros(nb, dtype=torch.uint8, pin_memory=True)
        self.ts_mu_base = None
        self.g_main = torch.cuda.Stream(device=self.dev)
        self.g_body = torch.cuda.Stream(device=self.dev)

    def project_step_dev(self, slot):
        """project_step with mu from the trial state (fp32 image of the fp64 mu)."""
        self.project_step(0.0, slot, mu_dev=self.ts.data_ptr() + 16)

    def _capture_iteration(self, config, carry):
        lib = self.lib
        rep = self.rep_hint_ready()
        g = ctypes.c_void_p()
        main, body = self.g_main, self.g_body
        main.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(main):
            _lib.check(lib.cbb_graph_capture_begin(main.cuda_stream, ctypes.byref(g)),
                       "cbb_graph_capture_begin")
            try:
                self.gradient()
                _lib.check(lib.cbb_trial_init(self.ts.data_ptr(), main.cuda_stream),
                           "cbb_trial_init")
                if rep:
                    self.rep_hint(0.0, mu_dev=self.ts.data_ptr() + 16)
                _lib.check(lib.cbb_graph_while_begin(g, body.cuda_stream), "while_begin")
                with torch.cuda.stream(body):
                    self.project_step_dev(1)
                    self.apply_norm2(self.dX, 2)
                    _lib.check(lib.cbb_trial_decide(g, self.ts.data_ptr(),
                                                    self.scal[1:2].data_ptr(),
                                                    self.scal[2:3].data_ptr(),
                                                    float(config.zeta),
                                                    int(config.max_shrink_per_iter)),
                               "cbb_trial_decide")
                _lib.check(lib.cbb_graph_while_end(g), "while_end")
                self.apply(self.Xn, self.AX)       # the accepted trial's iterate
                self.residual(0)
                if carry:
                    _lib.check(lib.cbb_trial_carry(self.ts.data_ptr(), main.cuda_stream),
                               "cbb_trial_carry")
                _lib.check(lib.cbb_graph_capture_end(g), "cbb_graph_capture_end")
            except Exception:
                lib.cbb_graph_destroy(g)
                raise
        torch.cuda.current_stream(self.dev).wait_stream(main)
        return g

    def graph_iteration(self, config, mu_base, carry):
        """Run one device-decided iteration.  Returns (new objective, mu, shrinks, fixed,
        collapsed)."""
        self._graph_setup()
        if mu_base != self.ts_mu_base:           # host mu_base (kappa, first use)
            hv = np.zeros(1, self._TS_DTYPE)
            hv["mu_base"] = mu_base
            raw = torch.from_numpy(hv.view(np.uint8).copy())
            self.ts[8:16].copy_(raw[8:16], non_blocking=False)
            self.ts_mu_base = mu_base
        key = (self.X.data_ptr(), carry)
        g = self._graphs.get(key)
        if g is None:
            g = self._graphs[key] = self._capture_iteration(config, carry)
        stream = torch.cuda.current_stream(self.dev)
        _lib.check(self.lib.cbb_graph_launch(g, stream.cuda_stream), "cbb_graph_launch")
        self.host[:1].copy_(self.scal[:1], non_blocking=True)
        self.ts_host.copy_(self.ts, non_blocking=True)
        stream.synchronize()
        t = self.ts_host.numpy()[:self._TS_DTYPE.itemsize].view(self._TS_DTYPE)[0]
        if carry:
            self.ts_mu_base = float(t["mu"])
        return (float(self.host[0]), float(t["mu"]), int(t["shrinks"]), bool(t["fixed"]),
                bool(t["status"]))

    def __del__(self):
        graphs = self.__dict__.get("_graphs") or {}
        for g in graphs.values():
            try:
                self.lib.cbb_graph_destroy(g)
            except Exception:
                pass
        graphs.clear()


_STAGE_BYTES = 256 << 20
_copy_pool = None


def _image_to_host(Xs: torch.Tensor, V: torch.Tensor = None) -> np.ndarray:
    """Image series X = Xs V^H (or Xs itself when V is None) -> (n, L) complex128 numpy (the
    reference's return type) without materialising it on the device: voxel chunks are
    decompressed and upcast on the GPU, copied into one of two reusable pinned staging buffers,
    and moved into the (pageable) result by host threads while the next chunk is copied."""
    global _copy_pool
    from concurrent.futures import ThreadPoolExecutor
    n = int(Xs.shape[0])
    L = int(Xs.shape[1]) if V is None else int(V.shape[0])
    out = np.empty((n, L), dtype=np.complex128)
    if n == 0 or L == 0:
        return out
    Vh = None if V is None else V.conj().transpose(0, 1)
    rows = max(1, min(n, _STAGE_BYTES // (16 * L)))
    bufs = [torch.empty((rows, L), dtype=torch.complex128, pin_memory=True) for _ in range(2)]
    if _copy_pool is None:
        _copy_pool = ThreadPoolExecutor(max_workers=8)
    pending = [[], []]
    stream = torch.cuda.current_stream(Xs.device)

    def drain(ev, src, dst):
        ev.synchronize()
        np.copyto(dst, src)

    for k, r0 in enumerate(range(0, n, rows)):
        b = k & 1
        for f in pending[b]:
            f.result()                     # the host copy out of this buffer has finished
        r1 = min(n, r0 + rows)
        blk = Xs[r0:r1] if Vh is None else Xs[r0:r1] @ Vh
        bufs[b][:r1 - r0].copy_(blk.to(torch.complex128), non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
        src = bufs[b].numpy()
        parts = np.linspace(0, r1 - r0, 9).astype(int)
        pending[b] = [_copy_pool.submit(drain, ev, src[a:c], out[r0 + a:r0 + c])
                      for a, c in zip(parts[:-1], parts[1:]) if c > a]
    for p in pending:
        for f in p:
            f.result()
    return out


def _ipg_loop(st, config, mu_base, y_norm, gt_t, gt_norm, n, d, on_iter=None):
    """The IPG iterations of solver.py:199-257 over a state object (``IpgState`` on one GPU,
    ``sharded.ShardedIpgState`` across ranks).  Returns (trace, have_proj)."""
    # X = 0: AX = 0, R = -w Y, obj = ||Y||_w^2
    st.residual(0)
    (obj,) = st.read(0)
    trace = SolveTrace()
    max_iters = 1 if config.mode == "tm" else config.max_iters
    start = time.perf_counter()
    trace.start = start
    have_proj = False
    graphs = hasattr(st, "graph_capable") and st.graph_capable(config)
    carry = config.step_policy == "carry_over"
    for k in range(1, max_iters + 1):
        t0 = time.perf_counter()
        if graphs and k >= 2:
            # device-decided iteration (gradient, trials, apply, residual in one graph)
            new_obj, mu, shrinks, fixed_pt, collapsed = st.graph_iteration(config, mu_base, carry)
            if collapsed:
                raise SolverError(
                    "step-size collapse: shrinkage exceeded "
                    f"{config.max_shrink_per_iter} sub-iterations")
            if on_iter is not None:
                on_iter(k, st, mu, shrinks, fixed_pt)
            if fixed_pt:
                break
            st.X, st.Xn = st.Xn, st.X
            st.idx, st.idx_n = st.idx_n, st.idx
            st.gam, st.gam_n = st.gam_n, st.gam
            have_proj = True
            if carry:
                mu_base = mu
            if not math.isfinite(new_obj):
                raise SolverError(f"non-finite fidelity at iteration {k}: {new_obj}")
            nmse = None
            if gt_t is not None:
                nmse = float(torch.linalg.vector_norm(st.decompress(st.X) - gt_t)) / gt_norm
            trace.add(iter=k, fidelity=math.sqrt(new_obj), mu=mu, shrinks=shrinks,
                      cost=n * d, nmse=nmse, seconds=time.perf_counter() - t0)
            if obj > 0.0 and (obj - new_obj) / obj < config.rel_tol:
                obj = new_obj
                break
            obj = new_obj
            if obj == 0.0:
                break
            continue
        st.gradient()
        if k == 1 and hasattr(st, "cold_hint"):
            st.cold_hint()                       # X = 0: warm-start atoms from the tile reps
        mu = mu_base
        shrinks = 0
        fixed_pt = False
        if k >= 2 and have_proj and hasattr(st, "rep_hint_ready") and st.rep_hint_ready():
            st.rep_hint(mu)                      # first trial: hint from the tile representatives
        while True:                              # step_shrinkage, solver.py:116-144
            st.project_step(mu, 1)
            if config.fixed_step is not None:
                (nd,) = st.read(1)
                fixed_pt = nd == 0.0
                break
            st.apply_norm2(st.dX, 2)
            nd, den = st.read(1, 2)
            if nd == 0.0:
                fixed_pt = True
                break
            ratio = math.inf if den == 0.0 else nd / den
            if mu <= ratio:
                break
            mu /= config.zeta
            shrinks += 1
            if shrinks > config.max_shrink_per_iter:
                raise SolverError(
                    "step-size collapse: shrinkage exceeded "
                    f"{config.max_shrink_per_iter} sub-iterations")
        if on_iter is not None:
            on_iter(k, st, mu, shrinks, fixed_pt)
        if fixed_pt:
            break
        st.X, st.Xn = st.Xn, st.X
        st.idx, st.idx_n = st.idx_n, st.idx
        st.gam, st.gam_n = st.gam_n, st.gam
        have_proj = True
        st.apply(st.X, st.AX)
        if k == 1 and config.fixed_step is None:   # kappa rescale, solver.py:220-230
            st.norm2(st.AX, 3)
            st.scaled_obj(1.0, 4)
            (e2, obj_x) = st.read(3, 4)
            e = math.sqrt(e2)
            if e > 0.0:
                kappa = y_norm / e
                st.scaled_obj(kappa, 5)
                (obj_k,) = st.read(5)
                if obj_k <= obj_x:
                    st.scale(st.X, kappa)
                    st.scale(st.AX, kappa)
                    st.gam.mul_(kappa)
                    mu_base *= kappa
        elif config.step_policy == "carry_over":
            mu_base = mu
        st.residual(0)
        (new_obj,) = st.read(0)
        if not math.isfinite(new_obj):
            raise SolverError(f"non-finite fidelity at iteration {k}: {new_obj}")
        nmse = None
        if gt_t is not None:
            nmse = float(torch.linalg.vector_norm(st.decompress(st.X) - gt_t)) / gt_norm
        trace.add(iter=k, fidelity=math.sqrt(new_obj), mu=mu, shrinks=shrinks, cost=n * d,
                  nmse=nmse, seconds=time.perf_counter() - t0)
        if obj > 0.0 and (obj - new_obj) / obj < config.rel_tol:
            obj = new_obj
            break
        obj = new_obj
        if obj == 0.0:
            break
    return trace, have_proj


_state_lock = threading.Lock()
_state_cache: dict = {}


def _state_for(Y, A, dictionary, basis, weights, dev):
    """The IPG state of a solve.  The most recent state is kept (with its captured iteration
    graphs) and reused by the next solve with the same operator, dictionary and basis objects:
    repeated solves (the reference's harness runs many) skip the buffer allocation and the graph
    capture.  The cache holds strong references, so the keyed ids cannot be recycled."""
    key = (dev.index, id(A), id(atoms_of(dictionary)), id(basis),
           None if basis is None else np.asarray(basis).shape, weights is None)
    with _state_lock:
        hit = _state_cache.get(key)
        if hit is not None and not hit[0].busy:
            st = hit[0]
            st.busy = True                # concurrent solves (harness threads) get their own
        else:
            st = None
            if hit is None:
                _state_cache.clear()      # one cached state: free the previous buffers
    if st is not None:
        st.load_measurements(Y, weights)
        st.reset_iterates()
        return st
    st = IpgState(Y, A, dictionary, basis, weights, dev)
    st.busy = True
    with _state_lock:
        if key not in _state_cache:
            _state_cache[key] = (st, A, atoms_of(dictionary), basis)
    return st


def _solve_core(Y, A, dictionary, tree, config, gt, basis, on_iter=None, return_device=False):
    """Device IPG loop following solver.py:155-257."""
    Ynp = np.asarray(Y)
    Ad = as_device_operator(A)
    dev = Ad.device
    weights = None
    if config.weights_enabled:
        if getattr(A, "weights", None) is None:
            raise SolverError("weights enabled but operator carries none")
        weights = np.asarray(A.weights, dtype=float)
    if config.mode == "coverblip" and tree is None:
        raise SolverError("coverblip mode needs a tree")
    with torch.cuda.device(dev):
        st = _state_for(Ynp, Ad, dictionary, basis, weights, dev)
        n, d = st.n, st.dd.d
        if config.fixed_step is not None:
            mu_base = config.fixed_step
        elif config.mu_init is not None:
            mu_base = config.mu_init
        else:
            mu_base = n / Ad.m
        y_norm = st.y_norm
        gt_t = None
        if gt is not None:
            gt_data = gt.data if hasattr(gt, "data") and not isinstance(gt, np.ndarray) else gt
            gt_t = torch.from_numpy(np.ascontiguousarray(gt_data, dtype=np.complex64)).to(dev)
            gt_norm = float(np.linalg.norm(gt_data))
        try:
            trace, have_proj = _ipg_loop(st, config, mu_base, y_norm, gt_t,
                                         gt_norm if gt_t is not None else None, n, d, on_iter)
            torch.cuda.current_stream(dev).synchronize()
            trace.total_time = time.perf_counter() - trace.start
            if return_device:             # the caller owns the state now: never reused
                with _state_lock:
                    for k_, v_ in list(_state_cache.items()):
                        if v_[0] is st:
                            del _state_cache[k_]
                return st, trace
            idx = st.idx.cpu().numpy().astype(np.int64) if have_proj else np.zeros(n, np.int64)
            gam = st.gam.cpu().numpy() if have_proj else np.zeros(n)
            maps = _maps_from(dictionary, idx, gam)
            out = _image_to_host(st.X, st.V)
            return out, maps, gam, trace
        finally:
            st.busy = False


def solve(Y, A, dictionary, tree, config: SolverConfig, gt=None, **kw):
    """solver.py:260-266: returns (image, maps, gammas, trace)."""
    if config.compressed is not None:
        raise SolverError("use solve_compressed for compressed configs")
    return _solve_core(Y, A, dictionary, tree, config, gt, basis=None, **kw)


def solve_compressed(Y, A, cdict, tree_s, config: SolverConfig, gt=None, **kw):
    """solver.py:269-275: iterates and searches in the s-dimensional subspace."""
    if config.compressed != cdict.s:
        raise SolverError("config.compressed does not match dictionary rank")
    return _solve_core(Y, A, cdict, tree_s, config, gt, basis=cdict.basis, **kw)
