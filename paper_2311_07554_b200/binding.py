"""ctypes binding of include/pacim.h — same names, argument marshalling only."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(HERE, "libpacim.so")

PACIM_P_CONST, PACIM_P_WIC, PACIM_P_UNIFORM = 0, 1, 2
PACIM_GEN_ER, PACIM_GEN_RMAT, PACIM_GEN_GRID = 0, 1, 2
STATUS = {0: "OK", -1: "EINVAL", -2: "ENOMEM", -3: "ECUDA", -4: "ENCCL", -5: "ESTATE",
          -6: "ENOTIMPL", -7: "ECHECK"}

# Every function declared in include/pacim.h (tests check the .so exports them).
EXPORTS = [
    "pacim_create", "pacim_destroy", "pacim_last_error", "pacim_version",
    "pacim_threshold_from_p", "pacim_threshold_uniform", "pacim_load_graph", "pacim_load_graph_async",
    "pacim_load_graph_upper", "pacim_load_graph_upper_async", "pacim_load_graph_device",
    "pacim_generate_graph", "pacim_graph_info", "pacim_get_graph",
    "pacim_build_sketches", "pacim_select_seeds", "pacim_gain0_to_device",
    "pacim_select_reset", "pacim_cover_local", "pacim_cover_local_sparse",
    "pacim_apply_deltas", "pacim_apply_dense", "pacim_clear_deltas", "pacim_argmax_device",
    "pacim_set_hash_rule", "pacim_simulate_ic", "pacim_set_selector",
    "pacim_get_gain0", "pacim_get_labels", "pacim_get_center_sketch",
    "pacim_get_stats", "pacim_nccl_unique_id", "pacim_init_comm",
]


class PacimError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class Stats(C.Structure):
    _fields_ = [
        ("n", C.c_uint32), ("m", C.c_uint64), ("R", C.c_uint32), ("R_local", C.c_uint32),
        ("rho", C.c_uint32), ("compressed", C.c_int), ("ncomp", C.c_uint64),
        ("nmember", C.c_uint64), ("live_pairs", C.c_uint64),
        ("t_build_ms", C.c_double), ("t_init_ms", C.c_double), ("t_edges_ms", C.c_double),
        ("t_compress_ms", C.c_double), ("t_compact_ms", C.c_double), ("t_gain_ms", C.c_double),
        ("t_centers_ms", C.c_double), ("t_select_ms", C.c_double),
        ("device_bytes", C.c_uint64), ("select_member_updates", C.c_uint64),
        ("select_bfs_visits", C.c_uint64), ("kernel_launches_build", C.c_uint32),
        ("kernel_launches_select", C.c_uint32), ("rows", C.c_uint32), ("nnonsingle", C.c_uint64),
        ("select_dense_steps", C.c_uint64), ("select_warp_slots", C.c_uint64),
        ("select_deferred_slots", C.c_uint64), ("select_row_items", C.c_uint64),
        ("select_chunk_items", C.c_uint64), ("select_inline_rows", C.c_uint64),
        ("select_edges", C.c_uint64), ("select_center_visits", C.c_uint64),
        ("select_center_found", C.c_uint64), ("batch_slots", C.c_uint32),
        ("select_evaluations", C.c_uint64), ("select_eval_rounds", C.c_uint64),
        ("hla_entries", C.c_uint64), ("hubs", C.c_uint32), ("select_hotsum_steps", C.c_uint64),
        ("lean", C.c_uint32), ("store", C.c_uint32), ("select_dist_replays", C.c_uint32),
        ("device_peak_bytes", C.c_uint64), ("select_celf_evaluations", C.c_uint64),
        ("build_hook_list", C.c_uint32),
    ]

    def asdict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None


def lib_path() -> str:
    return _LIB_PATH


def lib():
    """Load libpacim.so; raises if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} not built: run `python -m paper_2311_07554_b200.build`")
        L = C.CDLL(_LIB_PATH)
        P, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
        sig = {
            "pacim_create": (i32, [C.POINTER(P), i32, P, C.c_size_t, P]),
            "pacim_destroy": (None, [P]),
            "pacim_last_error": (C.c_char_p, [P]),
            "pacim_version": (C.c_char_p, []),
            "pacim_threshold_from_p": (u64, [C.c_double]),
            "pacim_threshold_uniform": (u64, [C.c_double, C.c_double]),
            "pacim_load_graph": (i32, [P, u32, u64, P, P, i32, u64, i32]),
            "pacim_load_graph_async": (i32, [P, u32, u64, P, P, i32, u64]),
            "pacim_load_graph_upper": (i32, [P, u32, u64, P, P, i32, u64, i32]),
            "pacim_load_graph_upper_async": (i32, [P, u32, u64, P, P, i32, u64]),
            "pacim_load_graph_device": (i32, [P, u32, u64, P, P, i32, u64, i32]),
            "pacim_generate_graph": (i32, [P, i32, P, i32, u64, i32, u64]),
            "pacim_graph_info": (i32, [P, P, P]),
            "pacim_get_graph": (i32, [P, P, P]),
            "pacim_build_sketches": (i32, [P, u32, u64, u64, u32, u32]),
            "pacim_select_seeds": (i32, [P, u32, P, P, P, P]),
            "pacim_gain0_to_device": (i32, [P, P]),
            "pacim_select_reset": (i32, [P]),
            "pacim_cover_local": (i32, [P, u32, P, P]),
            "pacim_cover_local_sparse": (i32, [P, u32, P, P, P, u64, P, P]),
            "pacim_apply_deltas": (i32, [P, P, P, P, u64, u32]),
            "pacim_set_hash_rule": (i32, [P, i32]),
            "pacim_simulate_ic": (i32, [P, P, u32, u32, u64, P]),
            "pacim_set_selector": (i32, [P, i32]),
            "pacim_apply_dense": (i32, [P, P, P, u32, u32]),
            "pacim_clear_deltas": (i32, [P, P, P, u64]),
            "pacim_argmax_device": (i32, [P, P, u32, P, P]),
            "pacim_get_gain0": (i32, [P, P]),
            "pacim_get_labels": (i32, [P, u32, P]),
            "pacim_get_center_sketch": (i32, [P, u32, P, P]),
            "pacim_get_stats": (i32, [P, C.POINTER(Stats)]),
            "pacim_nccl_unique_id": (i32, [P]),
            "pacim_init_comm": (i32, [P, i32, i32, P]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def pacim_threshold_from_p(p: float) -> int:
    return int(lib().pacim_threshold_from_p(float(p)))


def pacim_threshold_uniform(lo: float, hi: float) -> int:
    return int(lib().pacim_threshold_uniform(float(lo), float(hi)))


def pacim_nccl_unique_id() -> bytes:
    """A new 128-byte NCCL unique id (rank 0 creates it, every rank passes it to
    Context.pacim_init_comm)."""
    buf = C.create_string_buffer(128)
    rc = lib().pacim_nccl_unique_id(buf)
    if rc != 0:
        raise PacimError(rc, lib().pacim_last_error(None).decode())
    return buf.raw


def pacim_version() -> str:
    return lib().pacim_version().decode()


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _dptr(t) -> C.c_void_p:
    """Device pointer of a torch CUDA tensor (or an int address)."""
    return C.c_void_p(t if isinstance(t, int) else t.data_ptr())


class Context:
    """One pacim_ctx on one CUDA device (one per process/GPU)."""

    def __init__(self, device: int = 0, stream=None, workspace=None):
        """stream: a cudaStream_t (int) or a torch stream; default: torch's
        current stream on `device` (the legacy default stream is passed as
        cudaStreamLegacy), so library work is ordered with torch's work on the
        tensors it reads or writes (pacim_gain0_to_device, apply_*, ...).
        workspace: optional torch CUDA tensor (or (ptr, bytes)) the ctx
        carves all its device memory from (pacim_create's workspace)."""
        self._L = lib()
        h = C.c_void_p()
        if stream is None:
            try:
                import torch
                if torch.cuda.is_available():
                    stream = torch.cuda.current_stream(device).cuda_stream or 1  # 1: cudaStreamLegacy
            except ImportError:
                stream = None
        s = C.c_void_p(stream) if isinstance(stream, int) else (
            C.c_void_p(stream.cuda_stream or 1) if stream is not None else None)
        if workspace is None:
            wp, wb = None, 0
        elif isinstance(workspace, tuple):
            wp, wb = C.c_void_p(workspace[0]), int(workspace[1])
        else:
            wp, wb = C.c_void_p(workspace.data_ptr()), workspace.numel() * workspace.element_size()
        self._ws = workspace  # kept alive as long as the ctx
        rc = self._L.pacim_create(C.byref(h), int(device), wp, wb, s)
        if rc != 0:
            raise PacimError(rc, self._L.pacim_last_error(None).decode())
        self._h = h
        self.device = device

    def close(self):
        if getattr(self, "_h", None):
            self._L.pacim_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != 0:
            raise PacimError(rc, self._L.pacim_last_error(self._h).decode())

    def pacim_init_comm(self, rank: int, world: int, nccl_id: bytes):
        """NCCL communicator of this ctx (all ranks, same 128-byte id)."""
        assert len(nccl_id) == 128
        buf = C.create_string_buffer(bytes(nccl_id), 128)
        self._check(self._L.pacim_init_comm(self._h, int(rank), int(world), buf))

    # ------------------------------------------------------------- graph
    def pacim_load_graph(self, offsets: np.ndarray, neighbors: np.ndarray, pmodel: int, t32: int,
                         validate: int = 1):
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        nbr = np.ascontiguousarray(neighbors, dtype=np.uint32)
        self._check(self._L.pacim_load_graph(self._h, len(off) - 1, len(nbr), _ptr(off), _ptr(nbr),
                                             pmodel, t32, validate))

    def pacim_load_graph_async(self, offsets: np.ndarray, neighbors: np.ndarray, pmodel: int,
                               t32: int):
        """Enqueue the copy of a host CSR (pinned arrays overlap with compute);
        committed by the next pacim_build_sketches.  The arrays are
        kept referenced here until then (at most two loads pending)."""
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        nbr = np.ascontiguousarray(neighbors, dtype=np.uint32)
        self._check(self._L.pacim_load_graph_async(self._h, len(off) - 1, len(nbr), _ptr(off),
                                                   _ptr(nbr), pmodel, t32))
        self._staged = (getattr(self, "_staged", ()) + ((off, nbr),))[-3:]

    def pacim_load_graph_upper(self, uoffsets: np.ndarray, uneighbors: np.ndarray, pmodel: int,
                               t32: int, validate: int = 1):
        """Load from the upper CSR (each edge once, row u lists v > u sorted);
        the device builds the symmetric CSR."""
        off = np.ascontiguousarray(uoffsets, dtype=np.uint64)
        nbr = np.ascontiguousarray(uneighbors, dtype=np.uint32)
        self._check(self._L.pacim_load_graph_upper(self._h, len(off) - 1, len(nbr), _ptr(off),
                                                   _ptr(nbr), pmodel, t32, validate))

    def pacim_load_graph_upper_async(self, uoffsets: np.ndarray, uneighbors: np.ndarray,
                                     pmodel: int, t32: int):
        """Enqueue the copy of a host upper CSR (committed, and symmetrized on
        the device, by the next pacim_build_sketches); arrays kept referenced."""
        off = np.ascontiguousarray(uoffsets, dtype=np.uint64)
        nbr = np.ascontiguousarray(uneighbors, dtype=np.uint32)
        self._check(self._L.pacim_load_graph_upper_async(self._h, len(off) - 1, len(nbr),
                                                         _ptr(off), _ptr(nbr), pmodel, t32))
        self._staged = (getattr(self, "_staged", ()) + ((off, nbr),))[-3:]

    def pacim_load_graph_device(self, d_offsets, d_neighbors, n: int, nnz: int, pmodel: int,
                                t32: int, validate: int = 0):
        self._check(self._L.pacim_load_graph_device(self._h, n, nnz, _dptr(d_offsets),
                                                    _dptr(d_neighbors), pmodel, t32, validate))

    def pacim_generate_graph(self, kind: int, params, gen_seed: int, pmodel: int, t32: int):
        p = np.ascontiguousarray(params, dtype=np.uint64)
        self._check(self._L.pacim_generate_graph(self._h, kind, _ptr(p), len(p), gen_seed, pmodel,
                                                 t32))

    def pacim_graph_info(self):
        n, m = C.c_uint32(), C.c_uint64()
        self._check(self._L.pacim_graph_info(self._h, C.byref(n), C.byref(m)))
        return n.value, m.value

    def pacim_get_graph(self):
        n, m = self.pacim_graph_info()
        off = np.zeros(n + 1, np.uint64)
        nbr = np.zeros(2 * m, np.uint32)
        self._check(self._L.pacim_get_graph(self._h, _ptr(off), _ptr(nbr)))
        return off, nbr

    # ---------------------------------------------------------- sketches
    def pacim_simulate_ic(self, seeds, nsims: int, mc_seed: int) -> int:
        """Total vertices reached from `seeds` over nsims Monte-Carlo worlds (R21)."""
        s = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint32))
        t = C.c_uint64()
        self._check(self._L.pacim_simulate_ic(self._h, _ptr(s), len(s), int(nsims), int(mc_seed),
                                              C.byref(t)))
        return t.value

    def pacim_set_selector(self, selector: int):
        """0: incremental (default); 1: lazy, prefix doubling; 2: lazy, Win-Tree
        (NEXT f2; both lazy selectors count their evaluations)."""
        self._check(self._L.pacim_set_selector(self._h, int(selector)))

    def pacim_set_hash_rule(self, rule: int):
        """0: the paper's rule; 1: decorrelated (R20)."""
        self._check(self._L.pacim_set_hash_rule(self._h, int(rule)))

    def pacim_build_sketches(self, R: int, hash_seed: int, center_a32: int = 1 << 32,
                             shard_rank: int = 0, shard_world: int = 1):
        self._check(self._L.pacim_build_sketches(self._h, R, hash_seed, center_a32, shard_rank,
                                                 shard_world))

    def pacim_select_seeds(self, k: int):
        seeds = np.zeros(k, np.uint32)
        gain = np.zeros(k, np.int64)
        sig_num = np.zeros(k, np.int64)
        sigma = np.zeros(k, np.float64)
        self._check(self._L.pacim_select_seeds(self._h, k, _ptr(seeds), _ptr(gain), _ptr(sig_num),
                                               _ptr(sigma)))
        return seeds, gain, sig_num, sigma

    # ------------------------------------------------ multi-rank primitives
    def pacim_gain0_to_device(self, d_out):
        self._check(self._L.pacim_gain0_to_device(self._h, _dptr(d_out)))

    def pacim_select_reset(self):
        self._check(self._L.pacim_select_reset(self._h))

    def pacim_cover_local(self, s: int, d_delta) -> int:
        g = C.c_int64()
        self._check(self._L.pacim_cover_local(self._h, s, _dptr(d_delta), C.byref(g)))
        return g.value

    def pacim_cover_local_sparse(self, s: int, d_delta, d_list_v, d_list_d, cap: int):
        """-> (count, local_gain); count > cap means the list is incomplete."""
        g, c = C.c_int64(), C.c_uint64()
        self._check(self._L.pacim_cover_local_sparse(self._h, s, _dptr(d_delta), _dptr(d_list_v),
                                                     _dptr(d_list_d), cap, C.byref(c), C.byref(g)))
        return c.value, g.value

    def pacim_apply_deltas(self, d_gain, d_v, d_d, count: int, s: int = 0xFFFFFFFF):
        self._check(self._L.pacim_apply_deltas(self._h, _dptr(d_gain), _dptr(d_v), _dptr(d_d),
                                               count, s))

    def pacim_apply_dense(self, d_gain, d_delta, n: int, s: int = 0xFFFFFFFF):
        self._check(self._L.pacim_apply_dense(self._h, _dptr(d_gain), _dptr(d_delta), n, s))

    def pacim_clear_deltas(self, d_delta, d_v, count: int):
        self._check(self._L.pacim_clear_deltas(self._h, _dptr(d_delta), _dptr(d_v), count))

    def pacim_argmax_device(self, d_gain, n: int):
        s, g = C.c_uint32(), C.c_int64()
        self._check(self._L.pacim_argmax_device(self._h, _dptr(d_gain), n, C.byref(s), C.byref(g)))
        return s.value, g.value

    # -------------------------------------------------------- inspection
    def pacim_get_gain0(self):
        n, _ = self.pacim_graph_info()
        out = np.zeros(n, np.int64)
        self._check(self._L.pacim_get_gain0(self._h, _ptr(out)))
        return out

    def pacim_get_labels(self, r: int):
        n, _ = self.pacim_graph_info()
        out = np.zeros(n, np.uint32)
        self._check(self._L.pacim_get_labels(self._h, r, _ptr(out)))
        return out

    def pacim_get_center_sketch(self, r: int):
        rho = self.pacim_get_stats()["rho"]
        lab = np.zeros(max(rho, 1), np.uint32)
        sz = np.zeros(max(rho, 1), np.uint32)
        self._check(self._L.pacim_get_center_sketch(self._h, r, _ptr(lab), _ptr(sz)))
        return lab[:rho], sz[:rho]

    def pacim_get_stats(self) -> dict:
        return self.stats_raw().asdict()

    def stats_raw(self) -> "Stats":
        """pacim_get_stats into the ctypes struct itself (no dict): for timed loops."""
        s = Stats()
        self._check(self._L.pacim_get_stats(self._h, C.byref(s)))
        return s
