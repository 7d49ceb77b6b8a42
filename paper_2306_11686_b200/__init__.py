"""paper_2306_11686_b200 -- B200-native XSBench / RSBench macroscopic cross-section lookup.

Thin Python binding over the C ABI of ``include/gf_xs.h`` (``libgfxs.so``, sm_100a).  This module
only marshals arguments: every step of the lookup (grid build, sampling, sort, search,
interpolation, accumulation, hash) runs in the CUDA kernels behind the ABI.  PyTorch provides the
device memory, the current stream and (for multi-GPU) the process group.  There is no CPU
fallback: if the library cannot be loaded, or no sm_100a device is present, calls raise.

The method is the lookup loop GPU First runs on the GPU (Sec. 5.3.1); the
step-by-step readings are in DESIGN.md Sec. 3.
"""
from __future__ import annotations

import ctypes as C
import os

from .build import LIB as _LIB_PATH

__all__ = ["Params", "Grid", "PRGraph", "AMGMatrix", "verify", "lib", "XSBENCH", "RSBENCH", "NUCLIDE", "UNIONIZED", "HASH",
           "SORT_LOCALITY", "HISTORY", "HOST_IO", "HIST_WAVES", "HASH_MOD", "STARTING_SEED", "shard_range", "weak_range", "GFError"]

XSBENCH, RSBENCH = 0, 1
NUCLIDE, UNIONIZED, HASH = 0, 1, 2
SORT_LOCALITY, HISTORY, HOST_IO, HIST_WAVES = 1, 2, 4, 8
HASH_MOD = 999983
STARTING_SEED = 1070
ABI_VERSION = 1

ARR = dict(nuclide_grid=0, energy=1, unionized=2, index_grid=3, hash_grid=4, concs=5, mat_nucs=6, mat_offsets=7,
           thresholds=8, rs_poles=9, rs_pole_l=10, rs_windows=11, rs_K0RS=12, rs_pole_off=13, rs_win_off=14, union_bins=15,
           recip_width=16, intervals=17, nuclide_bins=18)

_STATUS = {0: "GF_OK", 1: "GF_E_INVAL", 2: "GF_E_NOMEM", 3: "GF_E_CUDA", 4: "GF_E_UNSUPPORTED", 5: "GF_E_MISMATCH"}


class GFError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class Params(C.Structure):
    _fields_ = [("abi_version", C.c_uint32), ("bench", C.c_int32), ("n_isotopes", C.c_int32),
                ("n_gridpoints", C.c_int64), ("grid_type", C.c_int32), ("hash_bins", C.c_int32),
                ("avg_n_poles", C.c_int32), ("avg_n_windows", C.c_int32), ("numL", C.c_int32),
                ("doppler", C.c_int32), ("init_seed", C.c_uint64), ("num_nucs", C.c_void_p),
                ("mats", C.c_void_p), ("max_num_nucs", C.c_int32), ("n_bands", C.c_int32), ("band", C.c_int32)]

    @classmethod
    def xsbench(cls, n_isotopes=355, n_gridpoints=11303, grid_type=UNIONIZED, hash_bins=10000, seed=42,
                n_bands=1, band=0):
        p = cls()
        _check(lib().gf_xs_default_params(XSBENCH, C.byref(p)))
        p.n_isotopes, p.n_gridpoints, p.grid_type, p.hash_bins, p.init_seed = (
            n_isotopes, n_gridpoints, grid_type, hash_bins, seed)
        p.n_bands, p.band = n_bands, band
        return p

    @classmethod
    def rsbench(cls, n_isotopes=355, avg_n_poles=1000, avg_n_windows=100, seed=42, doppler=1):
        p = cls()
        _check(lib().gf_xs_default_params(RSBENCH, C.byref(p)))
        p.n_isotopes, p.avg_n_poles, p.avg_n_windows, p.init_seed = n_isotopes, avg_n_poles, avg_n_windows, seed
        p.doppler = doppler
        return p


_lib = None


def lib():
    """Load libgfxs.so.  Fails loudly: there is no fallback path."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(nvcc, sm_100a).  There is no CPU fallback.")
        L = C.CDLL(_LIB_PATH)
        vp, u64, i32, sz = C.c_void_p, C.c_uint64, C.c_int32, C.c_size_t
        P = C.POINTER
        sig = {
            "gf_xs_default_params": (i32, [i32, vp]),
            "gf_xs_grid_bytes": (i32, [vp, P(sz), P(sz)]),
            "gf_xs_grid_init": (i32, [vp, C.c_int, vp, sz, vp, sz, vp, P(vp)]),
            "gf_xs_grid_free": (i32, [vp]),
            "gf_xs_grid_array": (i32, [vp, i32, P(vp), P(sz), P(C.c_int64)]),
            "gf_xs_batch_bytes": (i32, [vp, u64, C.c_uint32, P(sz)]),
            "gf_xs_batch_bytes_whole": (i32, [vp, u64, C.c_uint32, P(sz)]),
            "gf_xs_lookup_batch": (i32, [vp, u64, u64, u64, C.c_uint32, vp, vp, vp, sz, vp]),
            "gf_xs_lookup_batch_ev": (i32, [vp, u64, u64, u64, C.c_uint32, vp, vp, vp, sz, vp, vp]),
            "gf_xs_lookup_energies": (i32, [vp, vp, vp, u64, C.c_uint32, vp, vp, vp, sz, vp]),
            "gf_xs_lookup_energies_async": (i32, [vp, vp, vp, u64, C.c_uint32, vp, vp, sz, vp]),
            "gf_xs_history_bytes": (i32, [vp, u64, C.c_uint32, P(sz)]),
            "gf_xs_history_batch": (i32, [vp, u64, u64, i32, u64, C.c_uint32, vp, vp, vp, sz, vp]),
            "gf_xs_verify": (i32, [u64, u64, P(u64)]),
            "gf_xs_grid_info": (i32, [vp, P(i32)]),
            "gf_xs_debug_set_kernel": (i32, [vp, i32, u64, i32]),
            "gf_xs_kernel_for": (i32, [vp, u64, C.c_uint32, P(i32)]),
            "gf_xs_debug_set_division": (i32, [vp, i32]),
            "gf_xs_debug_set_prep_min": (i32, [vp, u64]),
            "gf_xs_selftest_div": (i32, [vp, vp, vp, vp, u64, vp]),
            "gf_xs_last_error": (C.c_char_p, []),
            "gf_pr_graph_bytes": (i32, [C.c_int64, i32, P(sz), P(sz)]),
            "gf_pr_graph_init": (i32, [C.c_int64, i32, u64, C.c_int, vp, sz, vp, sz, vp, P(vp)]),
            "gf_pr_graph_free": (i32, [vp]),
            "gf_pr_graph_info": (i32, [vp, P(C.c_int64), P(vp), P(vp), P(vp)]),
            "gf_pr_propagate": (i32, [vp, vp, vp, vp, vp]),
            "gf_pr_last_error": (C.c_char_p, []),
            "gf_amg_matrix_bytes": (i32, [i32, i32, i32, P(sz), P(C.c_int64)]),
            "gf_amg_matrix_init": (i32, [i32, i32, i32, C.c_int, vp, sz, vp, P(vp)]),
            "gf_amg_matrix_free": (i32, [vp]),
            "gf_amg_matrix_info": (i32, [vp, P(C.c_int64), P(C.c_int64), P(vp), P(vp), P(vp)]),
            "gf_amg_relax": (i32, [vp, vp, vp, vp, vp]),
            "gf_amg_last_error": (C.c_char_p, []),
            "gf_xs_version": (C.c_char_p, []),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def _check(status: int):
    if status != 0:
        raise GFError(status, lib().gf_xs_last_error().decode())


def verify(raw: int, expected: int | None = None) -> int:
    """hash = raw % 999983 (once, after all batches and shards: R-MOD).  Raises GFError(GF_E_INVAL)
    for a raw sum carrying the invalid-input flag (bit 63; gf_xs_lookup_energies)."""
    h = C.c_uint64()
    st = lib().gf_xs_verify(int(raw) & ((1 << 64) - 1), (1 << 64) - 1 if expected is None else int(expected),
                            C.byref(h))
    if st not in (0, 5):
        _check(st)
    if st == 5:
        raise GFError(5, lib().gf_xs_last_error().decode())
    return h.value


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Rank r of W takes the contiguous global indices [floor(r n / W), floor((r+1) n / W))."""
    lo, hi = (rank * n) // world, ((rank + 1) * n) // world
    return lo, hi - lo


def weak_range(n_per_rank: int, rank: int) -> tuple[int, int]:
    """Weak scaling: rank r takes the global indices [r n, (r+1) n) -- every rank does the config's
    single-GPU workload, the ranks' ranges are disjoint and consecutive, so the union over W ranks is
    the event batch [0, W n) and the all-reduced raw sum is that batch's."""
    return rank * n_per_rank, n_per_rank


def _stream_ptr(torch, stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


class Grid:
    """A grid built on the GPU (A0) into torch-owned device memory.

    ``Grid(Params.xsbench(...))`` or ``Grid(Params.rsbench(...))``.  The buffers stay alive as
    long as the object does; the handle is freed on ``close()`` / garbage collection.
    """

    def __init__(self, params: Params, device=None, stream=None, num_nucs=None, mats=None):
        import numpy as np
        import torch
        self.torch = torch
        self.params = params
        if num_nucs is not None:
            self._nn = np.ascontiguousarray(num_nucs, dtype=np.int32)
            self._mats = np.ascontiguousarray(mats, dtype=np.int32)
            params.num_nucs = self._nn.ctypes.data
            params.mats = self._mats.ctypes.data
            params.max_num_nucs = self._mats.shape[1]
        if device is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        elif isinstance(device, torch.device):
            dev = device if device.index is not None else torch.device("cuda", torch.cuda.current_device())
        else:
            dev = torch.device("cuda", int(device))
        self.device = dev
        gb, sb = C.c_size_t(), C.c_size_t()
        _check(lib().gf_xs_grid_bytes(C.byref(params), C.byref(gb), C.byref(sb)))
        self.grid_bytes = gb.value
        self.buf = torch.empty(gb.value, dtype=torch.uint8, device=dev)
        scratch = torch.empty(sb.value, dtype=torch.uint8, device=dev)
        h = C.c_void_p()
        with torch.cuda.device(dev):
            st = _stream_ptr(torch, stream)
            _check(lib().gf_xs_grid_init(C.byref(params), dev.index, C.c_void_p(self.buf.data_ptr()), gb.value,
                                         C.c_void_p(scratch.data_ptr()), sb.value, st, C.byref(h)))
            (stream or torch.cuda.current_stream()).synchronize()
        del scratch
        self.h = h
        self.bench = params.bench
        self.channels = 5 if params.bench == XSBENCH else 4
        self._scratch = {}  # one scratch buffer per CUDA stream (async calls on different streams must not share)

    @property
    def fastdiv(self) -> bool:
        v = C.c_int32()
        _check(lib().gf_xs_grid_info(self.h, C.byref(v)))
        return bool(v.value)

    KERNELS = {"auto": 0, "group": 1, "thread": 2, "tile": 4, "tilenb": 5, "warp": 6}

    def set_kernel(self, kern: str = "auto", tile_min: int = 0, nb: bool = True):
        """A/B and test hook (gf_xs_debug_set_kernel): force the sorted-path kernel of this grid."""
        _check(lib().gf_xs_debug_set_kernel(self.h, self.KERNELS[kern], tile_min, 1 if nb else 0))

    def set_prep_min(self, n: int = 1 << 23):
        """Test hook (gf_xs_debug_set_prep_min): batch size from which unionized tiles use per-tile indices."""
        _check(lib().gf_xs_debug_set_prep_min(self.h, n))

    def set_ieee_division(self, ieee: bool = True):
        """Test hook (gf_xs_debug_set_division): IEEE __ddiv_rn instead of the exact reciprocal scheme."""
        _check(lib().gf_xs_debug_set_division(self.h, 1 if ieee else 0))

    def kernel_for(self, n: int, flags: int = SORT_LOCALITY) -> str:
        """Name of the sorted-path kernel a batch of n lookups runs (gf_xs_kernel_for); "" if one kernel only."""
        k = C.c_int32()
        _check(lib().gf_xs_kernel_for(self.h, n, flags, C.byref(k)))
        return {v: name for name, v in self.KERNELS.items()}.get(k.value, "")

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            lib().gf_xs_grid_free(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ----------------------------------------------------------------- arrays (tests / tools)
    def array(self, name: str):
        """Device view (torch tensor) of one grid array; see gf_array in gf_xs.h for layouts."""
        torch = self.torch
        p, nb, pitch = C.c_void_p(), C.c_size_t(), C.c_int64()
        _check(lib().gf_xs_grid_array(self.h, ARR[name], C.byref(p), C.byref(nb), C.byref(pitch)))
        off = p.value - self.buf.data_ptr()
        raw = self.buf[off:off + nb.value]
        dt = {"nuclide_grid": torch.float64, "energy": torch.float64, "unionized": torch.float64,
              "index_grid": torch.int16, "hash_grid": torch.int16, "union_bins": torch.int32, "recip_width": torch.float64, "intervals": torch.float64, "nuclide_bins": torch.int16, "concs": torch.float64, "mat_nucs": torch.int32,
              "mat_offsets": torch.int32, "thresholds": torch.float64, "rs_poles": torch.float64,
              "rs_pole_l": torch.int32, "rs_windows": torch.float64, "rs_K0RS": torch.float64,
              "rs_pole_off": torch.int32, "rs_win_off": torch.int32}[name]
        if name == "hash_grid" and nb.value == self.params.n_isotopes * pitch.value * 4:
            dt = torch.int32  # u32 entries above 65536 gridpoints (XL / XXL)
        t = raw.view(dt)
        if dt == torch.int16:  # u16 interval indices (< n_gp <= 65536): widen without sign extension
            t = t.to(torch.int32) & 0xFFFF
        return t, pitch.value

    # ----------------------------------------------------------------- lookups
    def scratch_bytes(self, n: int, flags: int, whole: bool = False) -> int:
        """gf_xs_batch_bytes; whole=True: the larger size of the whole-batch host-I/O mode
        (gf_xs_batch_bytes_whole; host-I/O energies without per-lookup outputs)."""
        b = C.c_size_t()
        _check((lib().gf_xs_batch_bytes_whole if whole else lib().gf_xs_batch_bytes)(self.h, n, flags, C.byref(b)))
        return b.value

    def _get_scratch(self, need: int, stream=None):
        """The scratch buffer of `stream` (default: the current stream), grown to `need` bytes.  It is
        allocated on that stream, so the caching allocator reuses a replaced buffer only for work
        ordered after it on the same stream."""
        torch = self.torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        buf = self._scratch.get(s.cuda_stream)
        if buf is None or buf.numel() < need:
            with torch.cuda.stream(s):
                buf = torch.empty(max(need, 256), dtype=torch.uint8, device=self.device)
            self._scratch[s.cuda_stream] = buf
        return buf

    def lookup_batch_async(self, first: int, n: int, vsum, seed: int = STARTING_SEED, sort: bool = True,
                           macro_out=None, stream=None):
        """Enqueue lookups [first, first+n); ADDS sum(1+argmax) to the int64 device tensor `vsum`."""
        flags = SORT_LOCALITY if sort else 0
        sc = self._get_scratch(self.scratch_bytes(n, flags), stream)
        st = _stream_ptr(self.torch, stream)
        mo = C.c_void_p(macro_out.data_ptr()) if macro_out is not None else None
        _check(lib().gf_xs_lookup_batch(self.h, first, n, seed, flags, mo, C.c_void_p(vsum.data_ptr()),
                                        C.c_void_p(sc.data_ptr()), sc.numel(), st))

    def lookup_batch(self, first: int, n: int, seed: int = STARTING_SEED, sort: bool = True,
                     want_macro: bool = False, stream=None):
        """Lookups [first, first+n) -> raw sum (int), and the [n][5|4] fp64 macro xs if asked."""
        torch = self.torch
        vsum = torch.zeros(1, dtype=torch.int64, device=self.device)
        macro = torch.empty((n, self.channels), dtype=torch.float64, device=self.device) if want_macro else None
        self.lookup_batch_async(first, n, vsum, seed, sort, macro, stream)
        raw = int(vsum.item())
        return (raw, macro) if want_macro else raw

    def _check_states(self, E, mat, out, want_macro):
        """Argument checks of lookup_energies (marshalling only): dtypes, contiguity, sizes and devices
        must match what gf_xs_lookup_energies reads and writes, else ValueError (never a raw pointer
        into a wrong-sized or wrong-typed buffer)."""
        torch = self.torch
        if not isinstance(E, torch.Tensor) or not isinstance(mat, torch.Tensor):
            raise ValueError("E and mat must be torch tensors")
        if E.dtype != torch.float64 or mat.dtype != torch.uint8:
            raise ValueError(f"E must be float64 and mat uint8 (got {E.dtype}, {mat.dtype})")
        if E.dim() != 1 or mat.dim() != 1 or E.numel() != mat.numel():
            raise ValueError(f"E and mat must be 1-D of equal length (got {tuple(E.shape)}, {tuple(mat.shape)})")
        if not E.is_contiguous() or not mat.is_contiguous():
            raise ValueError("E and mat must be contiguous")
        if E.device != mat.device:
            raise ValueError(f"E and mat must be on the same device (got {E.device}, {mat.device})")
        if E.is_cuda and E.device != self.device:
            raise ValueError(f"device tensors must be on the grid's device {self.device} (got {E.device})")
        if out is not None:
            if not want_macro:
                raise ValueError("out given with want_macro=False")
            if (out.dtype != torch.float64 or tuple(out.shape) != (E.numel(), self.channels)
                    or not out.is_contiguous() or out.device != E.device):
                raise ValueError(f"out must be a contiguous float64 [{E.numel()}][{self.channels}] tensor on {E.device}")

    def lookup_energies(self, E, mat, sort: bool = True, want_macro: bool = True, stream=None, out=None):
        """Caller-supplied states (E float64 [n], mat uint8 [n]).  Device tensors -> device outputs;
        CPU tensors (pinned for speed) -> the call stages them (GF_HOST_IO, pipelined H2D / lookup /
        D2H) and returns host outputs.  `out`: an optional preallocated [n][5|4] fp64 output (pinned
        for host I/O) reused across calls.  Material ids > 11 or non-finite energies raise GFError
        (GF_E_INVAL; include/gf_xs.h)."""
        torch = self.torch
        self._check_states(E, mat, out, want_macro)
        n = E.numel()
        host = not E.is_cuda
        flags = (SORT_LOCALITY if sort else 0) | (HOST_IO if host else 0)
        st = _stream_ptr(torch, stream)
        if host:
            sc = self._get_scratch(self.scratch_bytes(n, flags, whole=not want_macro), stream)
            vs = C.c_uint64(0)
            macro = out
            if want_macro and macro is None:
                macro = torch.empty((n, self.channels), dtype=torch.float64, pin_memory=True)
            _check(lib().gf_xs_lookup_energies(self.h, C.c_void_p(E.data_ptr()), C.c_void_p(mat.data_ptr()), n, flags,
                                               C.c_void_p(macro.data_ptr()) if want_macro else None, C.byref(vs),
                                               C.c_void_p(sc.data_ptr()), sc.numel(), st))
            return (vs.value, macro) if want_macro else vs.value
        sc = self._get_scratch(self.scratch_bytes(n, flags), stream)
        vsum = torch.zeros(1, dtype=torch.int64, device=self.device)
        macro = out
        if want_macro and macro is None:
            macro = torch.empty((n, self.channels), dtype=torch.float64, device=self.device)
        _check(lib().gf_xs_lookup_energies(self.h, C.c_void_p(E.data_ptr()), C.c_void_p(mat.data_ptr()), n, flags,
                                           C.c_void_p(macro.data_ptr()) if want_macro else None,
                                           C.c_void_p(vsum.data_ptr()), C.c_void_p(sc.data_ptr()), sc.numel(), st))
        raw = int(vsum.item())
        if raw < 0:  # bit 63: the invalid-input flag
            raise GFError(1, "invalid caller inputs: material id > 11 or non-finite energy")
        return (raw, macro) if want_macro else raw

    def lookup_energies_async(self, E, mat, d_vsum, scratch, stream=None):
        """gf_xs_lookup_energies_async: pinned HOST E (float64 [n]) and mat (uint8 [n]) copied and looked up
        (sorted) on `stream` without waiting; the raw sum is ADDED to the device int64 tensor d_vsum[0].
        `scratch`: a device uint8 tensor of scratch_bytes(n, SORT_LOCALITY | HOST_IO, whole=True) bytes,
        not reused until the stream has passed this call (alternate two for back-to-back batches)."""
        torch = self.torch
        self._check_states(E, mat, None, False)
        if E.is_cuda or mat.is_cuda:
            raise ValueError("E and mat must be host tensors (pinned for asynchronous copies)")
        if d_vsum.device != self.device or d_vsum.dtype != torch.int64:
            raise ValueError("d_vsum must be an int64 tensor on the grid's device")
        if scratch.device != self.device or scratch.dtype != torch.uint8:
            raise ValueError("scratch must be a uint8 tensor on the grid's device")
        _check(lib().gf_xs_lookup_energies_async(self.h, C.c_void_p(E.data_ptr()), C.c_void_p(mat.data_ptr()),
                                                 E.numel(), SORT_LOCALITY, C.c_void_p(d_vsum.data_ptr()),
                                                 C.c_void_p(scratch.data_ptr()), scratch.numel(),
                                                 _stream_ptr(torch, stream)))

    # ----------------------------------------------------------------- history mode (NEXT-1)
    HIST_MODES = {"direct": 0, "waves": HIST_WAVES, "sorted": HIST_WAVES | SORT_LOCALITY}

    def history_batch_async(self, first_p: int, n_p: int, vsum, L: int = 34, seed: int = STARTING_SEED,
                            mode: str = "sorted", macro_out=None, stream=None):
        """Enqueue particles [first_p, first_p + n_p), L dependent lookups each (gf_xs_history_batch);
        ADDS the raw sum to the int64 device tensor `vsum`.  mode: "sorted" (waves + locality sort),
        "waves" or "direct" (one thread per particle)."""
        flags = self.HIST_MODES[mode]
        b = C.c_size_t()
        _check(lib().gf_xs_history_bytes(self.h, n_p, flags, C.byref(b)))
        sc = self._get_scratch(b.value, stream)
        mo = C.c_void_p(macro_out.data_ptr()) if macro_out is not None else None
        _check(lib().gf_xs_history_batch(self.h, first_p, n_p, L, seed, flags, mo, C.c_void_p(vsum.data_ptr()),
                                         C.c_void_p(sc.data_ptr()), sc.numel(), _stream_ptr(self.torch, stream)))

    def history_batch(self, first_p: int, n_p: int, L: int = 34, seed: int = STARTING_SEED, mode: str = "sorted",
                      want_macro: bool = False, stream=None):
        """History-based lookups -> raw sum (int), and the [n_p][L][5|4] fp64 macro xs if asked."""
        torch = self.torch
        vsum = torch.zeros(1, dtype=torch.int64, device=self.device)
        macro = torch.empty((n_p, L, self.channels), dtype=torch.float64, device=self.device) if want_macro else None
        self.history_batch_async(first_p, n_p, vsum, L, seed, mode, macro, stream)
        raw = int(vsum.item())
        return (raw, macro) if want_macro else raw


# ------------------------------------------------------------------ page-rank (NEXT-4, include/gf_pr.h)
def _pr_check(status: int):
    if status != 0:
        raise GFError(status, lib().gf_pr_last_error().decode())


class PRGraph:
    """Page-rank graph built on the GPU (readings R-PR-GRAPH / R-PR-STEP); ``propagate`` runs one step."""

    def __init__(self, n_nodes: int, avg_degree: int = 16, seed: int = 42, device=None, stream=None):
        import torch
        self.torch = torch
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else int(device))
        self.device, self.n = dev, n_nodes
        gb, sb = C.c_size_t(), C.c_size_t()
        _pr_check(lib().gf_pr_graph_bytes(n_nodes, avg_degree, C.byref(gb), C.byref(sb)))
        self.buf = torch.empty(gb.value, dtype=torch.uint8, device=dev)
        scratch = torch.empty(sb.value, dtype=torch.uint8, device=dev)
        h = C.c_void_p()
        with torch.cuda.device(dev):
            _pr_check(lib().gf_pr_graph_init(n_nodes, avg_degree, seed, dev.index, C.c_void_p(self.buf.data_ptr()),
                                             gb.value, C.c_void_p(scratch.data_ptr()), sb.value,
                                             _stream_ptr(torch, stream), C.byref(h)))
        del scratch
        self.h = h
        ne = C.c_int64()
        _pr_check(lib().gf_pr_graph_info(self.h, C.byref(ne), None, None, None))
        self.n_edges = ne.value
        self.contrib = torch.empty(n_nodes, dtype=torch.float64, device=dev)

    def arrays(self):
        """(rowptr u32 [N+1], col u32 [nnz], outdeg i32 [N]) as int64 CPU numpy arrays (tests)."""
        import numpy as np
        torch = self.torch
        rp, cl, od = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _pr_check(lib().gf_pr_graph_info(self.h, None, C.byref(rp), C.byref(cl), C.byref(od)))
        base = self.buf.data_ptr()

        def view(p, count, dt):
            off = p.value - base
            return self.buf[off:off + count * 4].view(dt).cpu().numpy()
        return (view(rp, self.n + 1, torch.int32).astype(np.int64) & 0xFFFFFFFF,
                view(cl, self.n_edges, torch.int32).astype(np.int64) & 0xFFFFFFFF, view(od, self.n, torch.int32))

    def propagate(self, r_in, r_out=None, stream=None):
        torch = self.torch
        if r_out is None:
            r_out = torch.empty_like(r_in)
        _pr_check(lib().gf_pr_propagate(self.h, C.c_void_p(r_in.data_ptr()), C.c_void_p(r_out.data_ptr()),
                                        C.c_void_p(self.contrib.data_ptr()), _stream_ptr(torch, stream)))
        return r_out

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            lib().gf_pr_graph_free(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ AMGmk relax (NEXT-4, include/gf_amg.h)
def _amg_check(status: int):
    if status != 0:
        raise GFError(status, lib().gf_amg_last_error().decode())


class AMGMatrix:
    """27-point Laplacian built on the GPU (R-AMG-MAT); ``relax`` runs one Jacobi sweep (R-AMG-RELAX)."""

    def __init__(self, nx: int, ny: int, nz: int, device=None, stream=None):
        import torch
        self.torch = torch
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else int(device))
        self.device, self.n = dev, nx * ny * nz
        b, nnz = C.c_size_t(), C.c_int64()
        _amg_check(lib().gf_amg_matrix_bytes(nx, ny, nz, C.byref(b), C.byref(nnz)))
        self.nnz = nnz.value
        self.buf = torch.empty(b.value, dtype=torch.uint8, device=dev)
        h = C.c_void_p()
        with torch.cuda.device(dev):
            _amg_check(lib().gf_amg_matrix_init(nx, ny, nz, dev.index, C.c_void_p(self.buf.data_ptr()), b.value,
                                                _stream_ptr(torch, stream), C.byref(h)))
            (stream or torch.cuda.current_stream()).synchronize()
        self.h = h

    def arrays(self):
        import numpy as np
        torch = self.torch
        rp, cl, vl = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _amg_check(lib().gf_amg_matrix_info(self.h, None, None, C.byref(rp), C.byref(cl), C.byref(vl)))
        base = self.buf.data_ptr()

        def view(p, nbytes, dt):
            off = p.value - base
            return self.buf[off:off + nbytes].view(dt).cpu().numpy()
        return (view(rp, (self.n + 1) * 4, torch.int32).astype(np.int64) & 0xFFFFFFFF,
                view(cl, self.nnz * 4, torch.int32).astype(np.int64) & 0xFFFFFFFF, view(vl, self.nnz * 8, torch.float64))

    def relax(self, f, u, out=None, stream=None):
        if out is None:
            out = self.torch.empty_like(u)
        _amg_check(lib().gf_amg_relax(self.h, C.c_void_p(f.data_ptr()), C.c_void_p(u.data_ptr()),
                                      C.c_void_p(out.data_ptr()), _stream_ptr(self.torch, stream)))
        return out

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            lib().gf_amg_matrix_free(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
