"""Parity oracle -- TEST INFRASTRUCTURE ONLY (never on the product path).

Two CPU implementations of the reference DPA-1 force path, behind one numpy API:

* ``Ref``  -- the UNMODIFIED reference C++ (/root/reference/proj) compiled from its own
  sources by ``oracle/Makefile`` into ``oracle/_ref/libnnmd_ref.so`` plus a C-ABI shim
  (``oracle/ref_capi.cpp``) over its public API.  Built in the dev container; the prebuilt
  .so travels to the GPU box.
* ``Port`` -- our own double-precision restatement (``oracle/dp_oracle.cpp``), each
  function citing the reference file:line it follows; pinned against ``Ref`` and the
  golden vectors in ``tests/golden/``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / reference
arm may import this package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libnnmd_ref.so")
PORT_SO = os.path.join(HERE, "_port", "libdp_oracle.so")

# Paper-sized DPA-1 spec: 1,584,945 parameters.
PAPER_SPEC = dict(rc=6.0, rcs=0.55 * 6.0, n_max=160, n_species=6, type_dim=8, n_feat=128,
                  n_reduced=32, n_attn=3, attn_dim=256, embed_hidden=(32, 64),
                  fit_hidden=(256, 256, 256))


def nmax_for_rc(rc: float) -> int:
    """n_max pinned per cutoff: 64 / 160 / 320 for rc = 4 / 6 / 8."""
    return {4.0: 64, 6.0: 160, 8.0: 320}.get(float(rc), 160)


def test_spec(rc, n_species=3, n_attn=3):
    """tests/support.hpp:49-64 test_model spec."""
    return dict(rc=rc, rcs=0.55 * rc, n_max=64, n_species=n_species, type_dim=4, n_feat=16,
                n_reduced=4, n_attn=n_attn, attn_dim=16, embed_hidden=(16,), fit_hidden=(32, 32))


def build(ref: bool = True) -> None:
    """Compile the oracle (port always; the reference only where /root/reference exists)."""
    targets = ["port"]
    if ref and os.path.isdir("/root/reference/proj"):
        targets += ["ref", "integration"]
    subprocess.run(["make", "-s", "-C", HERE, "-j8", *targets], check=True)


class OracleError(RuntimeError):
    pass


class CapacityError(OracleError):
    pass


_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_lp = C.POINTER(C.c_long)
_i64p = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)


def _d(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def _i(a):
    return a.ctypes.data_as(_ip) if a is not None else None


def _l(a):
    return a.ctypes.data_as(_lp) if a is not None else None


class _Lib:
    prefix = ""
    path = ""

    def __init__(self):
        if not os.path.exists(self.path):
            raise OracleError(f"oracle library missing: {self.path} (run make -C oracle)")
        self.lib = C.CDLL(self.path)
        L = self.lib
        p = self.prefix
        getattr(L, p + "last_error").restype = C.c_char_p
        getattr(L, p + "model_init").restype = C.c_void_p
        getattr(L, p + "model_init").argtypes = [C.c_double, C.c_double] + [C.c_int] * 7 + [_ip, C.c_int, _ip, C.c_int, C.c_uint64]
        getattr(L, p + "model_load").restype = C.c_void_p
        getattr(L, p + "model_load").argtypes = [C.c_char_p]
        getattr(L, p + "model_save").argtypes = [C.c_void_p, C.c_char_p]
        getattr(L, p + "model_free").argtypes = [C.c_void_p]
        getattr(L, p + "model_nparams").restype = C.c_long
        getattr(L, p + "model_nparams").argtypes = [C.c_void_p]

    def _chk(self, rc):
        if rc != 0:
            msg = getattr(self.lib, self.prefix + "last_error")().decode()
            raise (CapacityError if rc == 2 else OracleError)(msg)

    # -- model -------------------------------------------------------------------
    def model_init(self, spec: dict, seed: int = 1):
        eh = np.asarray(spec["embed_hidden"], dtype=np.int32)
        fh = np.asarray(spec["fit_hidden"], dtype=np.int32)
        h = getattr(self.lib, self.prefix + "model_init")(
            spec["rc"], spec["rcs"], spec["n_max"], spec["n_species"], spec["type_dim"],
            spec["n_feat"], spec["n_reduced"], spec["n_attn"], spec["attn_dim"], _i(eh), len(eh),
            _i(fh), len(fh), seed)
        if not h:
            self._chk(1)
        return h

    def model_load(self, path: str):
        h = getattr(self.lib, self.prefix + "model_load")(path.encode())
        if not h:
            self._chk(1)
        return h

    def model_save(self, h, path: str):
        self._chk(getattr(self.lib, self.prefix + "model_save")(h, path.encode()))

    def model_free(self, h):
        getattr(self.lib, self.prefix + "model_free")(h)

    def nparams(self, h) -> int:
        return getattr(self.lib, self.prefix + "model_nparams")(h)

    @staticmethod
    def _sys(pos, species, gids, box, periodic):
        pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
        species = np.ascontiguousarray(species, dtype=np.int32)
        gids = np.ascontiguousarray(np.arange(len(pos)) if gids is None else gids, dtype=np.int64)
        box = np.ascontiguousarray(box, dtype=np.float64)
        periodic = np.ascontiguousarray([1, 1, 1] if periodic is None else periodic, dtype=np.uint8)
        return pos, species, gids, box, periodic

    def _sysargs(self, pos, species, gids, box, periodic):
        return (len(pos), _d(pos), _i(species), gids.ctypes.data_as(_i64p), _d(box),
                periodic.ctypes.data_as(_u8p))


class Ref(_Lib):
    """The compiled reference (oracle/_ref/libnnmd_ref.so)."""
    prefix = "ref_"
    path = REF_SO

    def __init__(self):
        super().__init__()
        L = self.lib
        L.ref_model_set_nmax.argtypes = [C.c_void_p, C.c_int]
        L.ref_evaluate_dp.argtypes = [C.c_void_p, C.c_int, _dp, _ip, _i64p, _dp, _u8p, _dp, _dp, _dp, _dp]
        L.ref_center_rows.argtypes = [C.c_void_p, C.c_int, _dp, _ip, _i64p, _dp, _u8p, C.c_long, _ip, _ip, _ip, _dp, _lp]
        L.ref_dd_evaluate.argtypes = [C.c_void_p, C.c_int, _dp, _ip, _i64p, _dp, _u8p, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _ip, _lp]
        L.ref_build_halo.argtypes = [C.c_int, _dp, _dp, _u8p, _ip, C.c_int, C.c_double, C.c_long, _ip, _ip, _ip, _lp]
        L.ref_partition_ranks.argtypes = [_dp, C.c_int, C.c_double, _ip]
        L.ref_owner_ranks.argtypes = [C.c_int, _dp, _dp, _ip, _ip]
        L.ref_random_config.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_int, C.c_double, _dp, _dp, _ip]
        L.ref_make_dd_case.argtypes = [C.c_uint64, _dp, _dp, _ip, _ip, _dp]
        L.ref_time_centers.argtypes = [C.c_void_p, C.c_int, _dp, _ip, _i64p, _dp, _u8p, _ip, C.c_int, C.c_int, _dp, _dp, _dp]
        L.ref_fd_force_component.argtypes = [C.c_void_p, C.c_int, _dp, _ip, _i64p, _dp, _u8p, C.c_int, C.c_int, C.c_double, _dp]
        L.ref_evaluate_center_rows.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, _ip, _dp, _dp]
        L.ref_fit_throughput.argtypes = [C.c_int, _dp, _dp, _dp, _dp, _dp, _dp]
        L.ref_predict_throughput.argtypes = [C.c_double, C.c_double, C.c_double, _dp]
        L.ref_scaling_efficiency.argtypes = [C.c_int, _ip, _dp, C.c_int, C.c_int, _dp]
        L.ref_throughput_per_day.argtypes = [C.c_long, C.c_double, C.c_double, _dp]
        L.ref_evaluate_dp_mt.argtypes = [C.c_void_p, C.c_int, _dp, _ip, _i64p, _dp, _u8p, C.c_int, _dp, _dp, _dp, _dp]
        L.ref_step_slice.argtypes = [C.c_void_p, C.c_int, _dp, _ip, _i64p, _dp, _u8p, C.c_int, C.c_int, C.c_int,
                                     _dp, _dp, _dp]

    def set_nmax(self, h, n_max):
        self.lib.ref_model_set_nmax(h, n_max)

    def random_config(self, seed, n, density, n_species, min_sep=0.5):
        box = np.zeros(3)
        pos = np.zeros((n, 3))
        sp = np.zeros(n, dtype=np.int32)
        self._chk(self.lib.ref_random_config(seed, n, density, n_species, min_sep, _d(box), _d(pos), _i(sp)))
        return box, pos, sp

    def make_dd_case(self, seed):
        box = np.zeros(3)
        pos = np.zeros((256, 3))
        sp = np.zeros(256, dtype=np.int32)
        n = C.c_int()
        rc = C.c_double()
        self._chk(self.lib.ref_make_dd_case(seed, _d(box), _d(pos), _i(sp), C.byref(n), C.byref(rc)))
        return box, pos[: n.value].copy(), sp[: n.value].copy(), rc.value

    def evaluate(self, h, pos, species, box, gids=None, periodic=None, virial=True):
        pos, species, gids, box, periodic = self._sys(pos, species, gids, box, periodic)
        n = len(pos)
        e = C.c_double()
        f = np.zeros((n, 3))
        ae = np.zeros(n)
        w = np.zeros(9) if virial else None
        self._chk(self.lib.ref_evaluate_dp(h, *self._sysargs(pos, species, gids, box, periodic), C.byref(e), _d(f), _d(ae), _d(w)))
        return dict(energy=e.value, forces=f, atom_energy=ae, virial=None if w is None else w.reshape(3, 3))

    # -- analysis.cpp (Eq. 8 model, efficiencies) and engine.cpp throughput_per_day
    def fit_throughput(self, points):
        n = len(points)
        npa = np.ascontiguousarray([p[0] for p in points], dtype=np.float64)
        tra = np.ascontiguousarray([p[1] for p in points], dtype=np.float64)
        a, b, r2 = C.c_double(), C.c_double(), C.c_double()
        res = np.zeros(n)
        self._chk(self.lib.ref_fit_throughput(n, _d(npa), _d(tra), C.byref(a), C.byref(b), C.byref(r2), _d(res)))
        return {"alpha": a.value, "beta": b.value, "r_squared": r2.value, "residuals": list(res)}

    def predict_throughput(self, alpha, beta, n_p):
        out = C.c_double()
        self._chk(self.lib.ref_predict_throughput(alpha, beta, n_p, C.byref(out)))
        return out.value

    def scaling_efficiency(self, tr, reference, weak=False):
        keys = sorted(tr)
        npa = np.ascontiguousarray(keys, dtype=np.int32)
        tra = np.ascontiguousarray([tr[k] for k in keys], dtype=np.float64)
        eff = np.zeros(len(keys))
        self._chk(self.lib.ref_scaling_efficiency(len(keys), _i(npa), _d(tra), reference, int(weak), _d(eff)))
        return dict(zip(keys, eff.tolist()))

    def throughput_per_day(self, n_steps, dt, elapsed):
        out = C.c_double()
        self._chk(self.lib.ref_throughput_per_day(n_steps, dt, elapsed, C.byref(out)))
        return out.value

    def evaluate_mt(self, h, pos, species, box, workers, gids=None, periodic=None):
        """evaluate_dp on `workers` threads; bitwise equal to evaluate() (ref_capi.cpp)."""
        pos, species, gids, box, periodic = self._sys(pos, species, gids, box, periodic)
        n = len(pos)
        e = C.c_double()
        f = np.zeros((n, 3))
        ae = np.zeros(n)
        w = np.zeros(9)
        self._chk(self.lib.ref_evaluate_dp_mt(h, *self._sysargs(pos, species, gids, box, periodic), workers,
                                              C.byref(e), _d(f), _d(ae), _d(w)))
        return dict(energy=e.value, forces=f, atom_energy=ae, virial=w.reshape(3, 3))

    def step_slice(self, h, pos, species, box, c0, c1, workers, gids=None, periodic=None):
        """Reference per-step work for centres [c0, c1): build_neighbor_list + stock
        evaluate_dp with a LocalMask on `workers` threads.  -> (t_list s, t_eval s, E)."""
        pos, species, gids, box, periodic = self._sys(pos, species, gids, box, periodic)
        tl, te, es = C.c_double(), C.c_double(), C.c_double()
        self._chk(self.lib.ref_step_slice(h, *self._sysargs(pos, species, gids, box, periodic), c0, c1, workers,
                                          C.byref(tl), C.byref(te), C.byref(es)))
        return tl.value, te.value, es.value

    def center_rows(self, h, pos, species, box, gids=None, periodic=None, cap=None):
        pos, species, gids, box, periodic = self._sys(pos, species, gids, box, periodic)
        n = len(pos)
        cap = cap or n * 400
        counts = np.zeros(n, dtype=np.int32)
        mem = np.zeros(cap, dtype=np.int32)
        img = np.zeros((cap, 3), dtype=np.int32)
        d = np.zeros((cap, 3))
        tot = C.c_long()
        self._chk(self.lib.ref_center_rows(h, *self._sysargs(pos, species, gids, box, periodic), cap, _i(counts), _i(mem), _i(img), _d(d), C.byref(tot)))
        t = tot.value
        return counts, mem[:t].copy(), img[:t].copy(), d[:t].copy()

    def dd_evaluate(self, h, pos, species, box, n_ranks, scheme=0, workers=1, gids=None, periodic=None):
        pos, species, gids, box, periodic = self._sys(pos, species, gids, box, periodic)
        n = len(pos)
        e = C.c_double()
        f = np.zeros((n, 3))
        ae = np.zeros(n)
        dims = np.zeros(3, dtype=np.int32)
        stats = np.zeros((n_ranks, 4), dtype=np.int64)
        self._chk(self.lib.ref_dd_evaluate(h, *self._sysargs(pos, species, gids, box, periodic), n_ranks, scheme, workers,
                                           C.byref(e), _d(f), _d(ae), _i(dims), stats.ctypes.data_as(_lp)))
        return dict(energy=e.value, forces=f, atom_energy=ae, dims=dims, stats=stats)

    def partition_ranks(self, box, n_ranks, min_edge=0.0):
        dims = np.zeros(3, dtype=np.int32)
        self._chk(self.lib.ref_partition_ranks(_d(np.asarray(box, dtype=np.float64)), n_ranks, min_edge, _i(dims)))
        return dims

    def owner_ranks(self, pos, box, dims):
        pos = np.ascontiguousarray(pos, dtype=np.float64)
        out = np.zeros(len(pos), dtype=np.int32)
        self._chk(self.lib.ref_owner_ranks(len(pos), _d(pos), _d(np.asarray(box, dtype=np.float64)),
                                           _i(np.asarray(dims, dtype=np.int32)), _i(out)))
        return out

    def build_halo(self, pos, box, dims, rank, thickness, periodic=None):
        pos = np.ascontiguousarray(pos, dtype=np.float64)
        per = np.ascontiguousarray([1, 1, 1] if periodic is None else periodic, dtype=np.uint8)
        cap = 27 * len(pos)
        atom = np.zeros(cap, dtype=np.int32)
        own = np.zeros(cap, dtype=np.int32)
        sh = np.zeros((cap, 3), dtype=np.int32)
        nout = C.c_long()
        self._chk(self.lib.ref_build_halo(len(pos), _d(pos), _d(np.asarray(box, dtype=np.float64)), per.ctypes.data_as(_u8p),
                                          _i(np.asarray(dims, dtype=np.int32)), rank, thickness, cap, _i(atom), _i(own), _i(sh), C.byref(nout)))
        k = nout.value
        return atom[:k].copy(), own[:k].copy(), sh[:k].copy()

    def time_centers(self, h, pos, species, box, centers, workers, gids=None, periodic=None):
        pos, species, gids, box, periodic = self._sys(pos, species, gids, box, periodic)
        centers = np.ascontiguousarray(centers, dtype=np.int32)
        tl, tc, es = C.c_double(), C.c_double(), C.c_double()
        self._chk(self.lib.ref_time_centers(h, *self._sysargs(pos, species, gids, box, periodic), _i(centers), len(centers), workers,
                                            C.byref(tl), C.byref(tc), C.byref(es)))
        return tl.value, tc.value, es.value

    def fd_force(self, h, pos, species, box, atom, comp, hstep=1e-5, gids=None, periodic=None):
        pos, species, gids, box, periodic = self._sys(pos, species, gids, box, periodic)
        out = C.c_double()
        self._chk(self.lib.ref_fd_force_component(h, *self._sysargs(pos, species, gids, box, periodic), atom, comp, hstep, C.byref(out)))
        return out.value

    def evaluate_center(self, h, center_species, d, row_species):
        d = np.ascontiguousarray(d, dtype=np.float64).reshape(-1, 3)
        rs = np.ascontiguousarray(row_species, dtype=np.int32)
        e = C.c_double()
        g = np.zeros_like(d)
        self._chk(self.lib.ref_evaluate_center_rows(h, center_species, len(d), _d(d), _i(rs), C.byref(e), _d(g)))
        return e.value, g


class Port(_Lib):
    """Our CPU restatement (oracle/_port/libdp_oracle.so)."""
    prefix = "orc_"
    path = PORT_SO

    def __init__(self):
        super().__init__()
        L = self.lib
        L.orc_model_flat.argtypes = [C.c_void_p, _dp, C.c_long]
        L.orc_neighbor_rows.argtypes = [C.c_void_p, C.c_int, _dp, _ip, _i64p, _dp, _u8p, C.c_long, _ip, _ip, _ip, _dp, _lp]
        L.orc_evaluate.argtypes = [C.c_void_p, C.c_int, _dp, _ip, _i64p, _dp, _u8p, _dp, _dp, _dp, _dp]
        L.orc_evaluate_center.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, _ip, _dp, _dp]
        L.orc_partition_ranks.argtypes = [_dp, C.c_int, C.c_double, _ip]
        L.orc_owner_ranks.argtypes = [C.c_int, _dp, _dp, _ip, _ip]
        L.orc_build_halo.argtypes = [C.c_int, _dp, _dp, _u8p, _ip, C.c_int, C.c_double, C.c_long, _ip, _ip, _ip, _lp]
        L.orc_synth_system.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_uint64, _dp, _dp, _ip]
        L.orc_dd_rank.argtypes = [C.c_void_p, C.c_int, _dp, _ip, _i64p, _dp, _u8p, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _dp, _lp]

    def synth_system(self, n, rho=0.1, min_sep=0.9, seed=1):
        """Synthetic solvated-protein input (box, pos[n,3], species[n]); == nnmd_synth_system."""
        box = np.zeros(3)
        pos = np.zeros((n, 3))
        sp = np.zeros(n, dtype=np.int32)
        self._chk(self.lib.orc_synth_system(n, rho, min_sep, seed, _d(box), _d(pos), _i(sp)))
        return box, pos, sp

    def flat(self, h):
        n = self.nparams(h)
        out = np.zeros(n)
        self._chk(self.lib.orc_model_flat(h, _d(out), n))
        return out

    def neighbor_rows(self, h, pos, species, box, gids=None, periodic=None, cap=None):
        pos, species, gids, box, periodic = self._sys(pos, species, gids, box, periodic)
        n = len(pos)
        cap = cap or n * 400
        counts = np.zeros(n, dtype=np.int32)
        mem = np.zeros(cap, dtype=np.int32)
        img = np.zeros((cap, 3), dtype=np.int32)
        d = np.zeros((cap, 3))
        tot = C.c_long()
        self._chk(self.lib.orc_neighbor_rows(h, *self._sysargs(pos, species, gids, box, periodic), cap, _i(counts), _i(mem), _i(img), _d(d), C.byref(tot)))
        t = tot.value
        return counts, mem[:t].copy(), img[:t].copy(), d[:t].copy()

    def evaluate(self, h, pos, species, box, gids=None, periodic=None):
        pos, species, gids, box, periodic = self._sys(pos, species, gids, box, periodic)
        n = len(pos)
        e = C.c_double()
        f = np.zeros((n, 3))
        ae = np.zeros(n)
        w = np.zeros(9)
        self._chk(self.lib.orc_evaluate(h, *self._sysargs(pos, species, gids, box, periodic), C.byref(e), _d(f), _d(ae), _d(w)))
        return dict(energy=e.value, forces=f, atom_energy=ae, virial=w.reshape(3, 3))

    def evaluate_center(self, h, center_species, d, row_species):
        d = np.ascontiguousarray(d, dtype=np.float64).reshape(-1, 3)
        rs = np.ascontiguousarray(row_species, dtype=np.int32)
        e = C.c_double()
        g = np.zeros_like(d)
        self._chk(self.lib.orc_evaluate_center(h, center_species, len(d), _d(d), _i(rs), C.byref(e), _d(g)))
        return e.value, g

    def partition_ranks(self, box, n_ranks, min_edge=0.0):
        dims = np.zeros(3, dtype=np.int32)
        self._chk(self.lib.orc_partition_ranks(_d(np.asarray(box, dtype=np.float64)), n_ranks, min_edge, _i(dims)))
        return dims

    def owner_ranks(self, pos, box, dims):
        pos = np.ascontiguousarray(pos, dtype=np.float64)
        out = np.zeros(len(pos), dtype=np.int32)
        self._chk(self.lib.orc_owner_ranks(len(pos), _d(pos), _d(np.asarray(box, dtype=np.float64)),
                                           _i(np.asarray(dims, dtype=np.int32)), _i(out)))
        return out

    def build_halo(self, pos, box, dims, rank, thickness, periodic=None):
        pos = np.ascontiguousarray(pos, dtype=np.float64)
        per = np.ascontiguousarray([1, 1, 1] if periodic is None else periodic, dtype=np.uint8)
        cap = 27 * len(pos)
        atom = np.zeros(cap, dtype=np.int32)
        own = np.zeros(cap, dtype=np.int32)
        sh = np.zeros((cap, 3), dtype=np.int32)
        nout = C.c_long()
        self._chk(self.lib.orc_build_halo(len(pos), _d(pos), _d(np.asarray(box, dtype=np.float64)), per.ctypes.data_as(_u8p),
                                          _i(np.asarray(dims, dtype=np.int32)), rank, thickness, cap, _i(atom), _i(own), _i(sh), C.byref(nout)))
        k = nout.value
        return atom[:k].copy(), own[:k].copy(), sh[:k].copy()

    def dd_rank(self, h, pos, species, box, n_ranks, scheme, rank, gids=None, periodic=None):
        pos, species, gids, box, periodic = self._sys(pos, species, gids, box, periodic)
        n = len(pos)
        f = np.zeros((n, 3))
        ae = np.zeros(n)
        e = C.c_double()
        w = np.zeros(9)
        st = np.zeros(4, dtype=np.int64)
        self._chk(self.lib.orc_dd_rank(h, *self._sysargs(pos, species, gids, box, periodic), n_ranks, scheme, rank,
                                       _d(f), _d(ae), C.byref(e), _d(w), st.ctypes.data_as(_lp)))
        return dict(forces=f, atom_energy=ae, energy=e.value, virial=w.reshape(3, 3), stats=st[:3])
