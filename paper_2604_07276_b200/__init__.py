"""nnmd_b200 -- B200-native DPA-1 force path, drop-in for the nnmd NNPot/DeePMD backend.

Python mirror of the reference C++ interface (/root/reference/proj), over the C ABI of
``libnnmd_b200.so`` (``include/nnmd_b200.h``):

=========================  ==============================================================
here                        reference
=========================  ==============================================================
``ModelSpec``               ``nnmd::ModelSpec``            deeppot.hpp:63-75
``init_model``              ``nnmd::init_model``           deeppot.cpp:86-127 (bit-identical)
``load_model`` / ``save``   ``nnmd::load_model/save_model`` deeppot_io.cpp:56-160
``partition_ranks``         ``nnmd::partition_ranks``      decomp.cpp:17-57
``dd_evaluate``             ``nnmd::dd_evaluate``          decomp.cpp:265-542
``evaluate_dp``             ``nnmd::evaluate_dp`` (+ list) deeppot.cpp:315-369
``DpProvider``              ``nnmd::DpProvider``           engine.cpp:54-89
``Error/CapacityError``     ``nnmd::Error/CapacityError``  error.hpp:8-17
=========================  ==============================================================

Everything numeric runs in the CUDA library; there is no CPU fallback: importing works
without a GPU (host-only entry points such as model IO and ``partition_ranks``), but any
evaluation raises ``CudaError`` when no B200 is visible and ``ImportError`` when the
shared library has not been built (``python -c "import __graft_entry__ as g; g.build()"``).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libnnmd_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "nnmd_b200.h")

MASKED_REDUCTION = 0
WIDE_HALO = 1
PREC_FP32 = 0        # 3xTF32 tcgen05 (FP32-grade, 1e-5)
PREC_TF32 = 1        # 1xTF32 tcgen05 (stated tolerance 5e-3)
PREC_FP32_SIMT = 2   # FP32 FMA on CUDA cores (validation path)
TOLERANCE = {PREC_FP32: 1e-5, PREC_TF32: 5e-3, PREC_FP32_SIMT: 1e-5}


class Error(RuntimeError):
    """nnmd::Error"""


class CapacityError(Error):
    """nnmd::CapacityError (neighbour overflow, names the atom id)"""


class CudaError(Error):
    """CUDA / NCCL failure"""


def build(verbose: bool = False) -> str:
    """Compile libnnmd_b200.so for sm_100a (nvcc cross-compiles without a GPU)."""
    r = subprocess.run(["make", "-C", os.path.join(HERE, "csrc"), "-j8"], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nnmd_b200 build failed:\n" + r.stdout[-4000:] + r.stderr[-4000:])
    if verbose:
        print(r.stdout)
    return LIB_PATH


class _Spec(C.Structure):
    _fields_ = [("rc", C.c_double), ("rcs", C.c_double), ("n_max", C.c_int), ("n_species", C.c_int),
                ("type_dim", C.c_int), ("n_feat", C.c_int), ("n_reduced", C.c_int), ("n_attn", C.c_int),
                ("attn_dim", C.c_int), ("n_embed_hidden", C.c_int), ("embed_hidden", C.c_int * 8),
                ("n_fit_hidden", C.c_int), ("fit_hidden", C.c_int * 8)]


class _Opts(C.Structure):
    _fields_ = [("n_ranks", C.c_int), ("scheme", C.c_int), ("precision", C.c_int), ("device", C.c_int),
                ("world_size", C.c_int), ("world_rank", C.c_int), ("nccl_id", C.c_void_p)]


_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)
_lib = None


class _Span(C.Structure):
    _fields_ = [("rank", C.c_int), ("phase", C.c_int), ("t_start", C.c_double), ("t_end", C.c_double),
                ("step", C.c_long)]


class _Rec(C.Structure):
    _fields_ = [("step", C.c_long), ("kind", C.c_int), ("bytes", C.c_uint64), ("participants", C.c_int)]


PHASES = ("classical_md", "gather_positions", "dd_build", "neighbor_build", "inference", "ghost_force_route",
          "reduce_forces", "integrate")
COLLECTIVES = ("gather_positions", "ghost_force_route", "reduce_forces")


class _MdCfg(C.Structure):
    _fields_ = [("dt", C.c_double), ("n_steps", C.c_long), ("equil_steps", C.c_long),
                ("target_temperature", C.c_double), ("rescale_every", C.c_long)]


def lib():
    """The loaded libnnmd_b200.so (ImportError if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run paper_2604_07276_b200.build()")
    L = C.CDLL(LIB_PATH)
    L.nnmd_b200_last_error.restype = C.c_char_p
    L.nnmd_b200_version.restype = C.c_char_p
    L.nnmd_model_init.argtypes = [C.POINTER(_Spec), C.c_uint64, C.POINTER(C.c_void_p)]
    L.nnmd_model_load.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
    L.nnmd_model_save.argtypes = [C.c_void_p, C.c_char_p]
    L.nnmd_model_free.argtypes = [C.c_void_p]
    L.nnmd_model_nparams.argtypes = [C.c_void_p]
    L.nnmd_model_nparams.restype = C.c_long
    L.nnmd_model_get_spec.argtypes = [C.c_void_p, C.POINTER(_Spec)]
    L.nnmd_model_set_n_max.argtypes = [C.c_void_p, C.c_int]
    L.nnmd_partition_ranks.argtypes = [_dp, C.c_int, C.c_double, _ip]
    L.nnmd_route_schedule.argtypes = [C.c_int, C.c_int, C.c_int, _ip, C.c_void_p, C.c_int]
    L.nnmd_route_schedule.restype = C.c_int
    L.nnmd_b200_create.argtypes = [C.c_void_p, C.POINTER(_Opts), C.POINTER(C.c_void_p)]
    L.nnmd_b200_destroy.argtypes = [C.c_void_p]
    L.nnmd_b200_nccl_unique_id.argtypes = [C.c_void_p]
    L.nnmd_b200_compute.argtypes = [C.c_void_p, C.c_int64, _dp, _ip, _i64p, _dp, _u8p, _dp, _dp, _dp, _dp]
    L.nnmd_b200_compute_device.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, _dp, _u8p, C.c_void_p]
    L.nnmd_b200_run_md.argtypes = [C.c_void_p, C.c_int64, _dp, _dp, _dp, _ip, _i64p, _dp, _u8p,
                                   C.POINTER(_MdCfg), _dp, _dp]
    L.nnmd_b200_run_md_device.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_void_p, _dp, _u8p, C.POINTER(_MdCfg), C.c_void_p]
    L.nnmd_b200_set_trace.argtypes = [C.c_void_p, C.c_int, C.c_int]
    L.nnmd_b200_set_trace.restype = None
    L.nnmd_b200_set_step.argtypes = [C.c_void_p, C.c_long]
    L.nnmd_b200_set_step.restype = None
    L.nnmd_b200_trace_spans.argtypes = [C.c_void_p, C.POINTER(_Span), C.c_int]
    L.nnmd_b200_ledger.argtypes = [C.c_void_p, C.POINTER(_Rec), C.c_int]
    L.nnmd_b200_trace_clear.argtypes = [C.c_void_p]
    L.nnmd_b200_trace_clear.restype = None
    L.nnmd_b200_export_chrome_trace.argtypes = [C.c_void_p, C.c_char_p]
    L.nnmd_b200_rank_stats.argtypes = [C.c_void_p, C.c_int, _i64p, _dp]
    L.nnmd_b200_kernel_times.argtypes = [C.c_void_p, C.POINTER(C.c_char_p), _dp, C.c_int]
    L.nnmd_b200_set_debug.argtypes = [C.c_void_p, C.c_int]
    L.nnmd_b200_debug_nlist.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int), _ip, _ip, _ip, _ip]
    L.nnmd_b200_debug_ghosts.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int), _ip, _ip, _ip]
    L.nnmd_b200_stream.argtypes = [C.c_void_p]
    L.nnmd_b200_stream.restype = C.c_void_p
    L.nnmd_synth_system.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_uint64, _dp, _dp, _ip]
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().nnmd_b200_last_error().decode()
    raise {2: CapacityError, 3: CudaError}.get(rc, Error)(msg)


def _d(a):
    return a.ctypes.data_as(_dp) if a is not None else None


# ------------------------------------------------------------------------------ model
@dataclasses.dataclass
class ModelSpec:
    """nnmd::ModelSpec (deeppot.hpp:63-75); defaults = the paper-sized DPA-1."""
    rc: float = 6.0
    rcs: float = 3.3
    n_max: int = 160
    n_species: int = 6
    type_dim: int = 8
    n_feat: int = 128
    n_reduced: int = 32
    n_attn: int = 3
    attn_dim: int = 256
    embed_hidden: Sequence[int] = (32, 64)
    fit_hidden: Sequence[int] = (256, 256, 256)

    def to_c(self) -> _Spec:
        s = _Spec()
        for f in ("rc", "rcs", "n_max", "n_species", "type_dim", "n_feat", "n_reduced", "n_attn", "attn_dim"):
            setattr(s, f, getattr(self, f))
        s.n_embed_hidden = len(self.embed_hidden)
        for i, v in enumerate(self.embed_hidden):
            s.embed_hidden[i] = v
        s.n_fit_hidden = len(self.fit_hidden)
        for i, v in enumerate(self.fit_hidden):
            s.fit_hidden[i] = v
        return s


def paper_spec(rc: float = 6.0) -> ModelSpec:
    """Paper-sized DPA-1, 1,584,945 parameters; n_max 64/160/320 at rc 4/6/8."""
    return ModelSpec(rc=rc, rcs=0.55 * rc, n_max={4.0: 64, 6.0: 160, 8.0: 320}.get(float(rc), 160))


def test_spec(rc: float, n_species: int = 3, n_attn: int = 3) -> ModelSpec:
    """tests/support.hpp:49-64 test_model."""
    return ModelSpec(rc=rc, rcs=0.55 * rc, n_max=64, n_species=n_species, type_dim=4, n_feat=16,
                     n_reduced=4, n_attn=n_attn, attn_dim=16, embed_hidden=(16,), fit_hidden=(32, 32))


class DPModel:
    """Host-side model handle (nnmd::DPModel)."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.nnmd_model_free(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def n_params(self) -> int:
        return lib().nnmd_model_nparams(self._h)

    def spec(self) -> ModelSpec:
        s = _Spec()
        _check(lib().nnmd_model_get_spec(self._h, C.byref(s)))
        return ModelSpec(rc=s.rc, rcs=s.rcs, n_max=s.n_max, n_species=s.n_species, type_dim=s.type_dim,
                         n_feat=s.n_feat, n_reduced=s.n_reduced, n_attn=s.n_attn, attn_dim=s.attn_dim,
                         embed_hidden=tuple(s.embed_hidden[: s.n_embed_hidden]),
                         fit_hidden=tuple(s.fit_hidden[: s.n_fit_hidden]))

    def set_n_max(self, n_max: int) -> None:
        _check(lib().nnmd_model_set_n_max(self._h, n_max))

    def save(self, path: str) -> None:
        _check(lib().nnmd_model_save(self._h, path.encode()))


def init_model(spec: ModelSpec, seed: int = 1) -> DPModel:
    h = C.c_void_p()
    s = spec.to_c()
    _check(lib().nnmd_model_init(C.byref(s), seed, C.byref(h)))
    return DPModel(h.value)


def load_model(path: str) -> DPModel:
    h = C.c_void_p()
    _check(lib().nnmd_model_load(path.encode(), C.byref(h)))
    return DPModel(h.value)


def save_model(model: DPModel, path: str) -> None:
    model.save(path)


# ------------------------------------------------------------------------------ DD plan
def partition_ranks(box, n_ranks: int, min_edge: float = 0.0) -> np.ndarray:
    dims = np.zeros(3, dtype=np.int32)
    _check(lib().nnmd_partition_ranks(_d(np.asarray(box, dtype=np.float64)), n_ranks, min_edge,
                                      dims.ctypes.data_as(_ip)))
    return dims


class _RouteOp(C.Structure):
    _fields_ = [("kind", C.c_int), ("src", C.c_int), ("dst", C.c_int), ("peer", C.c_int),
                ("offset", C.c_long), ("count", C.c_int)]


def route_schedule(n_ranks: int, world_size: int, world_rank: int, counts) -> list:
    """Point-to-point plan of the ghost-force route for one process (host only; the plan
    the device path posts as one ncclGroupStart/End of ncclSend/ncclRecv).  counts[s, o] =
    routed entries from DD rank s to owner rank o.  Returns dicts {kind: "send"|"recv",
    src, dst, peer, offset, count} in posting order."""
    cnt = np.ascontiguousarray(np.asarray(counts, dtype=np.int32).reshape(n_ranks, n_ranks))
    cap = n_ranks * n_ranks
    ops = (_RouteOp * max(cap, 1))()
    k = lib().nnmd_route_schedule(n_ranks, world_size, world_rank, cnt.ctypes.data_as(_ip), ops, cap)
    if k < 0:
        raise Error(lib().nnmd_b200_last_error().decode())
    return [dict(kind="send" if o.kind == 0 else "recv", src=o.src, dst=o.dst, peer=o.peer, offset=o.offset,
                 count=o.count) for o in ops[:k]]


def synth_system(n: int, rho: float = 0.1, min_sep: float = 0.9, seed: int = 1):
    """Deterministic synthetic solvated protein (box, coords[n,3], species[n])."""
    box = np.zeros(3)
    pos = np.zeros((n, 3))
    sp = np.zeros(n, dtype=np.int32)
    _check(lib().nnmd_synth_system(n, rho, min_sep, seed, _d(box), _d(pos), sp.ctypes.data_as(_ip)))
    return box, pos, sp


# ------------------------------------------------------------------------------ device
class DeviceEvaluator:
    """One B200 context (streams, device weights, buffers, NCCL communicator)."""

    def __init__(self, model: DPModel, n_ranks: int = 1, scheme: int = MASKED_REDUCTION, device: int = 0,
                 world_size: int = 1, world_rank: int = 0, nccl_id: Optional[bytes] = None,
                 precision: int = PREC_FP32):
        o = _Opts()
        o.n_ranks, o.scheme, o.precision, o.device = n_ranks, scheme, precision, device
        o.world_size, o.world_rank = world_size, world_rank
        self._id = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        o.nccl_id = C.cast(self._id, C.c_void_p) if self._id is not None else None
        h = C.c_void_p()
        _check(lib().nnmd_b200_create(model.handle, C.byref(o), C.byref(h)))
        self._h = h
        self.n_ranks = n_ranks
        self.model = model

    def close(self):
        if getattr(self, "_h", None):
            lib().nnmd_b200_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib().nnmd_b200_nccl_unique_id(buf))
        return buf.raw

    def set_debug(self, on: bool = True) -> None:
        lib().nnmd_b200_set_debug(self._h, int(on))

    def compute(self, coords, types, box, gids=None, periodic=None, atom_energy=True):
        """Host buffers in, host results out (energy, forces[n,3], virial[3,3], atom_energy[n])."""
        coords = np.ascontiguousarray(coords, dtype=np.float64).reshape(-1, 3)
        types = np.ascontiguousarray(types, dtype=np.int32)
        n = len(coords)
        g = None if gids is None else np.ascontiguousarray(gids, dtype=np.int64)
        box = np.ascontiguousarray(box, dtype=np.float64)
        per = np.ascontiguousarray([1, 1, 1] if periodic is None else periodic, dtype=np.uint8)
        e = C.c_double()
        f = np.zeros((n, 3))
        w = np.zeros(9)
        ae = np.zeros(n) if atom_energy else None
        _check(lib().nnmd_b200_compute(self._h, n, _d(coords), types.ctypes.data_as(_ip),
                                       None if g is None else g.ctypes.data_as(_i64p), _d(box),
                                       per.ctypes.data_as(_u8p), C.byref(e), _d(f), _d(w), _d(ae)))
        return dict(energy=e.value, forces=f, virial=w.reshape(3, 3), atom_energy=ae)

    def run_md(self, coords, velocities, masses, types, box, dt, n_steps, gids=None, periodic=None,
               equil_steps=0, target_temperature=-1.0, rescale_every=10):
        """Device-resident MD loop (run_md, engine.cpp:143-211).  coords/velocities
        (float64 [n,3], C-contiguous) are updated in place; returns (potential[n_steps],
        total[n_steps])."""
        for a in (coords, velocities):
            if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous):
                raise Error("run_md: coords and velocities must be C-contiguous float64 arrays")
        n = len(coords)
        masses = np.ascontiguousarray(masses, dtype=np.float64)
        types = np.ascontiguousarray(types, dtype=np.int32)
        g = None if gids is None else np.ascontiguousarray(gids, dtype=np.int64)
        box = np.ascontiguousarray(box, dtype=np.float64)
        per = np.ascontiguousarray([1, 1, 1] if periodic is None else periodic, dtype=np.uint8)
        cfg = _MdCfg(dt, n_steps, equil_steps, target_temperature, rescale_every)
        pot = np.zeros(max(n_steps, 1))
        tot = np.zeros(max(n_steps, 1))
        _check(lib().nnmd_b200_run_md(self._h, n, _d(coords), _d(velocities), _d(masses), types.ctypes.data_as(_ip),
                                      None if g is None else g.ctypes.data_as(_i64p), _d(box),
                                      per.ctypes.data_as(_u8p), C.byref(cfg), _d(pot), _d(tot)))
        return pot[:n_steps], tot[:n_steps]

    def run_md_device(self, n: int, d_coords: int, d_vel: int, d_mass: int, d_types: int, d_gids: int, box,
                      dt, n_steps, d_energies: int, periodic=None, equil_steps=0, target_temperature=-1.0,
                      rescale_every=10):
        """Device pointers; d_energies[2k] = potential, [2k+1] = total energy of step k."""
        box = np.ascontiguousarray(box, dtype=np.float64)
        per = np.ascontiguousarray([1, 1, 1] if periodic is None else periodic, dtype=np.uint8)
        cfg = _MdCfg(dt, n_steps, equil_steps, target_temperature, rescale_every)
        _check(lib().nnmd_b200_run_md_device(self._h, n, C.c_void_p(d_coords), C.c_void_p(d_vel),
                                             C.c_void_p(d_mass), C.c_void_p(d_types), C.c_void_p(d_gids), _d(box),
                                             per.ctypes.data_as(_u8p), C.byref(cfg), C.c_void_p(d_energies)))

    # ---- TraceSink / CollectiveLedger (trace.hpp, decomp.hpp:64-107)
    def set_trace(self, spans: bool = True, ledger: bool = True) -> None:
        lib().nnmd_b200_set_trace(self._h, int(spans), int(ledger))

    def set_step(self, step: int) -> None:
        lib().nnmd_b200_set_step(self._h, step)

    def trace_spans(self):
        """[(rank, phase_name, t_start, t_end, step)] recorded since the last clear."""
        n = lib().nnmd_b200_trace_spans(self._h, None, 0)
        buf = (_Span * max(n, 1))()
        lib().nnmd_b200_trace_spans(self._h, buf, n)
        return [(s.rank, PHASES[s.phase], s.t_start, s.t_end, s.step) for s in buf[:n]]

    def ledger(self):
        """[(step, kind_name, bytes, participants)] recorded since the last clear."""
        n = lib().nnmd_b200_ledger(self._h, None, 0)
        buf = (_Rec * max(n, 1))()
        lib().nnmd_b200_ledger(self._h, buf, n)
        return [(r.step, COLLECTIVES[r.kind], int(r.bytes), r.participants) for r in buf[:n]]

    def clear_trace(self) -> None:
        lib().nnmd_b200_trace_clear(self._h)

    def export_chrome_trace(self, path: str) -> None:
        _check(lib().nnmd_b200_export_chrome_trace(self._h, path.encode()))

    def compute_device(self, n: int, d_coords: int, d_types: int, d_gids: int, box, d_out: int, periodic=None):
        """Device pointers in/out; d_out = [E, W(9), F(3n), ae(n)] float64."""
        box = np.ascontiguousarray(box, dtype=np.float64)
        per = np.ascontiguousarray([1, 1, 1] if periodic is None else periodic, dtype=np.uint8)
        _check(lib().nnmd_b200_compute_device(self._h, n, C.c_void_p(d_coords), C.c_void_p(d_types),
                                              C.c_void_p(d_gids), _d(box), per.ctypes.data_as(_u8p),
                                              C.c_void_p(d_out)))

    def stream(self) -> int:
        return lib().nnmd_b200_stream(self._h) or 0

    def rank_stats(self, rank: int):
        counts = np.zeros(4, dtype=np.int64)
        ms = np.zeros(4)
        _check(lib().nnmd_b200_rank_stats(self._h, rank, counts.ctypes.data_as(_i64p), _d(ms)))
        return dict(locals=int(counts[0]), ghosts=int(counts[1]), centers=int(counts[2]),
                    route_entries=int(counts[3]), dd_ms=ms[0], neighbor_ms=ms[1], inference_ms=ms[2],
                    comm_ms=ms[3])

    def kernel_times(self):
        n = lib().nnmd_b200_kernel_times(self._h, None, None, 0)
        names = (C.c_char_p * max(n, 1))()
        ms = np.zeros(max(n, 1))
        k = lib().nnmd_b200_kernel_times(self._h, names, _d(ms), n)
        return [(names[i].decode(), float(ms[i])) for i in range(k)]

    def debug_nlist(self, rank: int, n_max: int):
        nc = C.c_int()
        _check(lib().nnmd_b200_debug_nlist(self._h, rank, C.byref(nc), None, None, None, None))
        c = nc.value
        ca = np.zeros(c, dtype=np.int32)
        idx = np.zeros(c * n_max, dtype=np.int32)
        img = np.zeros(c * n_max * 3, dtype=np.int32)
        cnt = np.zeros(c, dtype=np.int32)
        _check(lib().nnmd_b200_debug_nlist(self._h, rank, C.byref(nc), ca.ctypes.data_as(_ip), idx.ctypes.data_as(_ip),
                                           img.ctypes.data_as(_ip), cnt.ctypes.data_as(_ip)))
        return ca, idx.reshape(c, n_max), img.reshape(c, n_max, 3), cnt

    def debug_ghosts(self, rank: int):
        ng = C.c_int()
        _check(lib().nnmd_b200_debug_ghosts(self._h, rank, C.byref(ng), None, None, None))
        g = ng.value
        atom = np.zeros(g, dtype=np.int32)
        own = np.zeros(g, dtype=np.int32)
        sh = np.zeros(g * 3, dtype=np.int32)
        _check(lib().nnmd_b200_debug_ghosts(self._h, rank, C.byref(ng), atom.ctypes.data_as(_ip), own.ctypes.data_as(_ip),
                                            sh.ctypes.data_as(_ip)))
        return atom, own, sh.reshape(g, 3)


# ------------------------------------------------------------------------------ reference-shaped API
@dataclasses.dataclass
class SimBox:
    lengths: Sequence[float]
    periodic: Sequence[bool] = (True, True, True)


@dataclasses.dataclass
class AtomSet:
    global_ids: np.ndarray
    species: np.ndarray
    positions: np.ndarray
    velocities: Optional[np.ndarray] = None
    masses: Optional[np.ndarray] = None

    def __len__(self):
        return len(self.positions)


@dataclasses.dataclass
class DdResult:
    energy: float
    forces: np.ndarray
    atom_energy: np.ndarray
    virial: np.ndarray
    grid: np.ndarray
    stats: list


_eval_cache = {}


def dd_evaluate(atoms: AtomSet, box: SimBox, model: DPModel, n_ranks: int, scheme: int = MASKED_REDUCTION,
                device: int = 0) -> DdResult:
    """nnmd::dd_evaluate on one B200 (all DD ranks on this device, ascending order)."""
    key = (id(model), n_ranks, scheme, device)
    ev = _eval_cache.get(key)
    if ev is None or ev.model is not model:
        ev = _eval_cache[key] = DeviceEvaluator(model, n_ranks=n_ranks, scheme=scheme, device=device)
    r = ev.compute(atoms.positions, atoms.species, box.lengths, gids=atoms.global_ids,
                   periodic=[int(p) for p in box.periodic])
    thick = model.spec().rc * (1 if scheme == MASKED_REDUCTION else 2)
    grid = partition_ranks(box.lengths, n_ranks, thick)
    return DdResult(r["energy"], r["forces"], r["atom_energy"], r["virial"], grid,
                    [ev.rank_stats(k) for k in range(n_ranks)])


def evaluate_dp(atoms: AtomSet, box: SimBox, model: DPModel, device: int = 0) -> DdResult:
    """Single-domain evaluation (one DD rank reproduces evaluate_dp's rows bit for bit)."""
    return dd_evaluate(atoms, box, model, 1, MASKED_REDUCTION, device)


@dataclasses.dataclass
class StepContext:
    step: int = 0


@dataclasses.dataclass
class ProviderResult:
    energy: float
    forces: np.ndarray
    virial: Optional[np.ndarray] = None


class ForceProvider:
    """nnmd::ForceProvider (engine.hpp:28-34)."""

    def name(self) -> str:
        raise NotImplementedError

    def evaluate(self, atoms: AtomSet, box: SimBox, ctx: StepContext) -> ProviderResult:
        raise NotImplementedError


class DpProvider(ForceProvider):
    """nnmd::DpProvider (engine.hpp:51-74, engine.cpp:54-89) on B200.

    Options mirror DpProvider::Options: decomposed, scheme, n_ranks, species_map; the
    group mask selects the NN atoms (others get zero force)."""

    @dataclasses.dataclass
    class Options:
        decomposed: bool = False
        scheme: int = WIDE_HALO
        n_ranks: int = 1
        workers: int = 1  # accepted for API parity; device ranks replace host workers
        species_map: Sequence[int] = ()
        device: int = 0

    def __init__(self, model: DPModel, opts: "DpProvider.Options" = None, group_mask=None):
        self.model = model
        self.opts = opts or DpProvider.Options()
        self.group = None if group_mask is None or len(group_mask) == 0 else np.asarray(group_mask, dtype=bool)
        nr = self.opts.n_ranks if self.opts.decomposed else 1
        sch = self.opts.scheme if self.opts.decomposed else MASKED_REDUCTION
        self._ev = DeviceEvaluator(model, n_ranks=nr, scheme=sch, device=self.opts.device)

    def name(self) -> str:
        return "dp_dd" if self.opts.decomposed else "dp_single"

    def evaluate(self, atoms: AtomSet, box: SimBox, ctx: StepContext = None) -> ProviderResult:
        idx = np.arange(len(atoms)) if self.group is None else np.nonzero(self.group)[0]
        sp = np.asarray(atoms.species, dtype=np.int32)[idx]
        if len(self.opts.species_map):
            smap = np.asarray(self.opts.species_map, dtype=np.int32)
            if np.any(sp < 0) or np.any(sp >= len(smap)):
                raise Error("DpProvider: species outside the species map")
            sp = smap[sp]
        forces = np.zeros((len(atoms), 3))
        if len(idx) == 0:
            return ProviderResult(0.0, forces, np.zeros((3, 3)))
        r = self._ev.compute(np.asarray(atoms.positions)[idx], sp, box.lengths,
                             gids=np.asarray(atoms.global_ids)[idx], periodic=[int(p) for p in box.periodic])
        forces[idx] = r["forces"]
        return ProviderResult(r["energy"], forces, r["virial"])


@dataclasses.dataclass
class MDConfig:
    """nnmd::MDConfig (engine.hpp:99-107)."""
    dt: float = 0.002
    n_steps: int = 0
    output_every: int = 0  # trajectory cadence (file output is out of scope here)
    equil_steps: int = 0
    target_temperature: float = -1.0
    rescale_every: int = 10


@dataclasses.dataclass
class RunSummary:
    """nnmd::RunSummary (engine.hpp:109-117)."""
    steps: int
    dt: float
    elapsed_seconds: float
    throughput: float
    potential_energy: np.ndarray
    total_energy: np.ndarray


def run_md(atoms: AtomSet, box: SimBox, config: MDConfig, provider: "DpProvider") -> RunSummary:
    """nnmd::run_md (engine.cpp:143-211) with one DpProvider, on the device: positions and
    velocities stay in HBM for the whole run.  atoms.positions / atoms.velocities are
    updated in place."""
    import time
    if config.dt <= 0:
        raise Error("run_md: dt must be > 0")
    if config.n_steps < 0:
        raise Error("run_md: n_steps must be >= 0")
    if provider.group is not None or len(provider.opts.species_map):
        raise Error("run_md (device loop): group masks and species maps need the host loop")
    pos = np.ascontiguousarray(atoms.positions, dtype=np.float64)
    vel = np.ascontiguousarray(atoms.velocities, dtype=np.float64)
    t0 = time.perf_counter()
    pot, tot = provider._ev.run_md(pos, vel, atoms.masses, atoms.species, box.lengths, config.dt, config.n_steps,
                                   gids=atoms.global_ids, periodic=[int(p) for p in box.periodic],
                                   equil_steps=config.equil_steps, target_temperature=config.target_temperature,
                                   rescale_every=config.rescale_every)
    el = time.perf_counter() - t0
    atoms.positions[...] = pos
    atoms.velocities[...] = vel
    thr = config.n_steps * config.dt / el * 86400.0 if el > 0 else 0.0
    return RunSummary(config.n_steps, config.dt, el, thr, pot, tot)


def header_functions() -> list:
    """Names of all functions declared in include/nnmd_b200.h (for the export test)."""
    import re
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(nnmd_\w+)\s*\(", txt)))
