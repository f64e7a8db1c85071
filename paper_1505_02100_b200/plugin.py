"""Thin ctypes binding of libplugin.so (include/plugin.h).  Argument marshalling only:
every step of the method runs in the library's CUDA kernels.  There is no CPU
fallback: if the library or a CUDA device is missing, calls raise.

Tensors are torch tensors (torch is used for device memory and streams only).
Function names match the C ABI.
"""
from __future__ import annotations

import ctypes
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
DEFAULT_LIB = os.path.join(HERE, "libplugin.so")
LIB_PATH = os.environ.get("PLUGIN_LIB_PATH") or DEFAULT_LIB

PLUGIN_OK, PLUGIN_E_INVALID, PLUGIN_E_NONFINITE, PLUGIN_E_DEGENERATE, PLUGIN_E_DOMAIN, PLUGIN_E_CUDA = range(6)
STATUS_NAMES = {0: "PLUGIN_OK", 1: "PLUGIN_E_INVALID", 2: "PLUGIN_E_NONFINITE", 3: "PLUGIN_E_DEGENERATE",
                4: "PLUGIN_E_DOMAIN", 5: "PLUGIN_E_CUDA"}


class PluginError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class plugin_result(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("path", ctypes.c_int32), ("n", ctypes.c_int64)] + [
        (k, ctypes.c_double) for k in ("mean", "var", "sigma", "psi8_ns", "g1", "psi6", "g2", "psi4", "h",
                                       "g1_z", "psi6_z", "g2_z", "psi4_z", "h_z", "S6", "S4")]

    def to_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


DPI_MAX_STAGES = 5


class plugin_dpi_result(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("stages", ctypes.c_int32), ("n", ctypes.c_int64),
                ("mean", ctypes.c_double), ("var", ctypes.c_double), ("sigma", ctypes.c_double),
                ("psi_ns_z", ctypes.c_double)] + [
        (k, ctypes.c_double * DPI_MAX_STAGES) for k in ("g_z", "g", "psi_z", "psi")] + [
        ("h_z", ctypes.c_double), ("h", ctypes.c_double)]

    def to_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_}
        for k in ("g_z", "g", "psi_z", "psi"):   # stage j -> value (j = 1..stages)
            d[k] = {j: d[k][j - 1] for j in range(1, self.stages + 1)}
        return d


class plugin_fx128(ctypes.Structure):
    _fields_ = [("limb", ctypes.c_int64 * 4)]


RESULT_BYTES = ctypes.sizeof(plugin_result)
_lib = None


def lib():
    """Load libplugin.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        P, i64, i32, sz, d = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t, ctypes.c_double
        sig = {
            "plugin_workspace_bytes": (sz, [i64]),
            "plugin_host_workspace_bytes": (sz, [i64]),
            "plugin_h": (i32, [P, i64, P, P, sz, P]),
            "plugin_h_ex": (i32, [P, i64, P, ctypes.c_uint, P, sz, P]),
            "plugin_h_sync": (i32, [P, i64, P, P, sz, P]),
            "plugin_h_batch": (i32, [P, P, i32, P, ctypes.c_uint, P]),
            "plugin_graph_create": (i32, [P, i64, P, P, sz, ctypes.c_uint, ctypes.POINTER(P)]),
            "plugin_graph_launch": (i32, [P, P]),
            "plugin_graph_destroy": (None, [P]),
            "plugin_h_host": (i32, [P, i64, P, P, sz, P]),
            "psi_r": (i32, [P, i64, d, i32, P, P, sz, P]),
            "plugin_step1": (i32, [P, i64, P, P, sz, P]),
            "psi_r_shard": (i32, [i64, i32, i32, i32, P, P, P, sz, P]),
            "plugin_after_psi6": (i32, [P, P, P]),
            "plugin_after_psi4": (i32, [P, P, P]),
            "plugin_num_tiles": (i64, [i64, i32]),
            "plugin_tile_edge": (i64, [i64, i32]),
            "plugin_work_item": (i32, [i64, i32, i64, ctypes.POINTER(i64)]),
            "psi_r_shard_g": (i32, [i64, d, i32, i32, i32, P, P, sz, P]),
            "plugin_prepare": (i32, [P, i64, P, sz, P]),
            "plugin_psi_from_total": (i32, [P, i64, d, i32, P, P]),
            "plugin_shard_tiles": (None, [i64, i32, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]),
            "plugin_dpi": (i32, [P, i64, i32, P, P, sz, P]),
            "plugin_sort": (i32, [P, i64, P, P, sz, P]),
            "plugin_q32_workspace_bytes": (sz, [i64]),
            "psi_r_q32": (i32, [P, i64, i64, i32, P, P, sz, P]),
            "plugin_h_q32": (i32, [P, i64, P, P, sz, P]),
            "kde_workspace_bytes": (sz, [i64, i64]),
            "kde_eval": (i32, [P, i64, d, P, i64, P, P, sz, P]),
            "kde_prepare": (i32, [P, i64, P, sz, P]),
            "kde_eval_prepared": (i32, [i64, d, P, i64, P, P, sz, P]),
            "plugin_last_error": (ctypes.c_char_p, []),
            "plugin_version": (ctypes.c_char_p, []),
        }
        for name, (res, args) in sig.items():
            if LIB_PATH != DEFAULT_LIB and not hasattr(L, name):
                continue  # an A/B variant library (PLUGIN_LIB_PATH) built from an older source
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


PLUGIN_SKIP_UNDERFLOW = 1
PLUGIN_MULTI_KERNEL = 2
PLUGIN_PATH_GROUPED = 1  # plugin_result["path"] bit: the exact grouped fp64 pass ran (group.cu)

EXPORTED = ("plugin_workspace_bytes", "plugin_host_workspace_bytes", "plugin_h", "plugin_h_ex", "plugin_h_batch",
            "plugin_graph_create", "plugin_graph_launch", "plugin_graph_destroy",
            "plugin_h_sync", "plugin_h_host",
            "psi_r", "plugin_step1", "psi_r_shard", "plugin_after_psi6", "plugin_after_psi4", "plugin_num_tiles",
            "plugin_shard_tiles", "plugin_tile_edge", "plugin_work_item", "psi_r_shard_g", "plugin_prepare",
            "plugin_psi_from_total", "plugin_dpi", "plugin_sort", "plugin_q32_workspace_bytes", "psi_r_q32", "plugin_h_q32",
            "kde_workspace_bytes", "kde_eval", "kde_prepare",
            "kde_eval_prepared", "plugin_last_error", "plugin_version")


def _check(st: int):
    if st == PLUGIN_E_INVALID or st == PLUGIN_E_CUDA:
        raise PluginError(st, lib().plugin_last_error().decode())
    return st


def _dev(t: torch.Tensor) -> torch.device:
    """The device of a tensor argument (checked like _x, without copying)."""
    if not (isinstance(t, torch.Tensor) and t.is_cuda):
        raise TypeError("expected a CUDA tensor")
    return t.device


class _On:
    """Run a library call on the device of its input and on `stream` (None: that device's
    current stream; a torch.cuda.Stream; or a raw cudaStream_t handle).  Inside the block the
    device and the stream are current, so temporaries (workspace, contiguous copies, outputs)
    are allocated for that stream and the caching allocator cannot hand them out again while
    the library's kernels on it still use them."""

    def __init__(self, device, stream=None):
        self.device = torch.device(device)
        if stream is None:
            self.stream = torch.cuda.current_stream(self.device)
        elif isinstance(stream, torch.cuda.Stream):
            self.stream = stream
        else:
            self.stream = torch.cuda.ExternalStream(int(stream), device=self.device)

    def __enter__(self):
        self._dev = torch.cuda.device(self.device)
        self._dev.__enter__()
        self._st = torch.cuda.stream(self.stream)
        self._st.__enter__()
        return self

    def __exit__(self, *exc):
        self._st.__exit__(*exc)
        self._dev.__exit__(*exc)
        return False

    @property
    def handle(self):
        return ctypes.c_void_p(self.stream.cuda_stream)

    def uses(self, *tensors):
        """Mark caller-owned inputs as used on this stream (Tensor.record_stream): the caching
        allocator then keeps their memory until the library's kernels on it have run, even if
        the caller drops its last reference right after the (asynchronous) call."""
        for t in tensors:
            if isinstance(t, torch.Tensor) and t.is_cuda:
                t.record_stream(self.stream)


def _x(x: torch.Tensor) -> torch.Tensor:
    if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float32 and x.dim() == 1):
        raise TypeError("x must be a 1-D CUDA float32 tensor")
    return x.contiguous()


def plugin_workspace_bytes(n: int) -> int:
    return lib().plugin_workspace_bytes(n)


def plugin_host_workspace_bytes(n: int) -> int:
    return lib().plugin_host_workspace_bytes(n)


def workspace(n: int, device=None, host: bool = False) -> torch.Tensor:
    """A 256-byte aligned uint8 device buffer of the size the library needs."""
    nbytes = plugin_host_workspace_bytes(n) if host else plugin_workspace_bytes(n)
    t = torch.empty(nbytes + 256, dtype=torch.uint8, device=device or "cuda")
    off = (-t.data_ptr()) % 256
    return t[off:off + nbytes]


def new_result(device=None) -> torch.Tensor:
    return torch.empty(RESULT_BYTES, dtype=torch.uint8, device=device or "cuda")


def read_result(buf: torch.Tensor) -> dict:
    """Copy a device plugin_result to the host (synchronises) and decode it."""
    h = buf.detach().to("cpu").numpy().tobytes()
    return plugin_result.from_buffer_copy(h).to_dict()


def plugin_h(x: torch.Tensor, out: torch.Tensor | None = None, ws: torch.Tensor | None = None, stream=None,
             flags: int = 0):
    """Alg. 1 on the device (asynchronous).  Returns the device result buffer.
    ``flags``: PLUGIN_SKIP_UNDERFLOW (bit-identical result, less work; plugin_h_ex)."""
    with _On(_dev(x), stream) as on:
        x = _x(x)
        on.uses(x)
        n = x.numel()
        ws = workspace(n, x.device) if ws is None else ws
        out = new_result(x.device) if out is None else out
        _check(lib().plugin_h_ex(x.data_ptr(), n, out.data_ptr(), int(flags), ws.data_ptr(), ws.numel(), on.handle))
    return out


def plugin_h_batch(x: torch.Tensor, offsets: torch.Tensor, out: torch.Tensor | None = None, stream=None,
                   flags: int = 0) -> torch.Tensor:
    """Alg. 1 for every sample x[offsets[b]:offsets[b+1]] (2 <= n_b <= 2048), one CTA each
    (T = 256 tiles: agrees with plugin_h to fp32 rounding); returns the device buffer of count
    plugin_result records (read_results decodes it)."""
    if not (isinstance(offsets, torch.Tensor) and offsets.is_cuda and offsets.dtype == torch.int64):
        raise TypeError("offsets must be a CUDA int64 tensor of count + 1 entries")
    with _On(_dev(x), stream) as on:
        x = _x(x)
        on.uses(x)
        offsets = offsets.contiguous()
        count = offsets.numel() - 1
        out = torch.empty(max(count, 1) * RESULT_BYTES, dtype=torch.uint8, device=x.device) if out is None else out
        _check(lib().plugin_h_batch(x.data_ptr(), offsets.data_ptr(), count, out.data_ptr(), int(flags), on.handle))
    return out


class PluginGraph:
    """plugin_h on fixed buffers as a CUDA graph (plugin_graph_create / _launch / _destroy):
    refill x in place, call launch(), read the result buffer."""

    def __init__(self, x: torch.Tensor, out: torch.Tensor | None = None, ws: torch.Tensor | None = None,
                 flags: int = 0):
        self.handle = None
        self.x = _x(x)
        self.device = self.x.device
        with torch.cuda.device(self.device):
            n = self.x.numel()
            self.ws = workspace(n, self.device) if ws is None else ws
            self.out = new_result(self.device) if out is None else out
            h = ctypes.c_void_p()
            _check(lib().plugin_graph_create(self.x.data_ptr(), n, self.out.data_ptr(), self.ws.data_ptr(),
                                             self.ws.numel(), int(flags), ctypes.byref(h)))
        self.handle = h

    def launch(self, stream=None) -> torch.Tensor:
        # no temporaries here: only the stream needs resolving (kept light: latency path)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        h = stream.cuda_stream if isinstance(stream, torch.cuda.Stream) else int(stream)
        _check(lib().plugin_graph_launch(self.handle, ctypes.c_void_p(h)))
        return self.out

    def close(self):
        if self.handle:
            lib().plugin_graph_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def read_results(buf: torch.Tensor, count: int) -> list[dict]:
    h = buf.detach().to("cpu").numpy().tobytes()
    return [plugin_result.from_buffer_copy(h[k * RESULT_BYTES:(k + 1) * RESULT_BYTES]).to_dict() for k in range(count)]


def plugin_h_sync(x: torch.Tensor, ws: torch.Tensor | None = None, stream=None) -> dict:
    with _On(_dev(x), stream) as on:
        x = _x(x)
        on.uses(x)
        n = x.numel()
        ws = workspace(n, x.device) if ws is None else ws
        res = plugin_result()
        _check(lib().plugin_h_sync(x.data_ptr(), n, ctypes.addressof(res), ws.data_ptr(), ws.numel(), on.handle))
    return res.to_dict()


def plugin_h_host(x_host: torch.Tensor, ws: torch.Tensor | None = None, stream=None) -> dict:
    """End to end from host memory (copies inside the call)."""
    if not (isinstance(x_host, torch.Tensor) and not x_host.is_cuda and x_host.dtype == torch.float32):
        raise TypeError("x_host must be a CPU float32 tensor (pinned for best speed)")
    x_host = x_host.contiguous()
    n = x_host.numel()
    dev = ws.device if ws is not None else torch.device("cuda", torch.cuda.current_device())
    with _On(dev, stream) as on:
        ws = workspace(n, dev, host=True) if ws is None else ws
        res = plugin_result()
        _check(lib().plugin_h_host(x_host.data_ptr(), n, ctypes.addressof(res), ws.data_ptr(), ws.numel(), on.handle))
    return res.to_dict()


def psi_r(x: torch.Tensor, g: float, r: int, out: torch.Tensor | None = None, ws: torch.Tensor | None = None,
          stream=None) -> torch.Tensor:
    """Psi_r(g) (Steps IV/VI) as a device float64[1] tensor (asynchronous)."""
    with _On(_dev(x), stream) as on:
        x = _x(x)
        on.uses(x)
        n = x.numel()
        ws = workspace(n, x.device) if ws is None else ws
        out = torch.empty(1, dtype=torch.float64, device=x.device) if out is None else out
        _check(lib().psi_r(x.data_ptr(), n, float(g), int(r), out.data_ptr(), ws.data_ptr(), ws.numel(), on.handle))
    return out


def plugin_step1(x: torch.Tensor, out: torch.Tensor, ws: torch.Tensor, stream=None):
    with _On(_dev(x), stream) as on:
        x = _x(x)
        on.uses(x)
        _check(lib().plugin_step1(x.data_ptr(), x.numel(), out.data_ptr(), ws.data_ptr(), ws.numel(), on.handle))
    return out


def new_partial(device=None) -> torch.Tensor:
    return torch.empty(4, dtype=torch.int64, device=device or "cuda")


def psi_r_shard(n: int, r: int, rank: int, world: int, out: torch.Tensor, partial: torch.Tensor, ws: torch.Tensor,
                stream=None):
    with _On(ws.device, stream) as on:
        _check(lib().psi_r_shard(n, r, rank, world, out.data_ptr(), partial.data_ptr(), ws.data_ptr(), ws.numel(),
                                 on.handle))
    return partial


def plugin_prepare(x: torch.Tensor, ws: torch.Tensor, stream=None) -> torch.Tensor:
    """Sort X into the workspace, Step I and the distinct-value count (for psi_r_shard_g)."""
    with _On(_dev(x), stream) as on:
        x = _x(x)
        on.uses(x)
        _check(lib().plugin_prepare(x.data_ptr(), x.numel(), ws.data_ptr(), ws.numel(), on.handle))
    return ws


def psi_r_shard_g(n: int, g: float, r: int, rank: int, world: int, partial: torch.Tensor, ws: torch.Tensor,
                  stream=None) -> torch.Tensor:
    """This rank's share of Psi_r at a host bandwidth g, as 4 fixed-point limbs (int64[4])."""
    with _On(ws.device, stream) as on:
        _check(lib().psi_r_shard_g(int(n), float(g), int(r), int(rank), int(world), partial.data_ptr(),
                                   ws.data_ptr(), ws.numel(), on.handle))
    return partial


def plugin_psi_from_total(total: torch.Tensor, n: int, g: float, r: int, out: torch.Tensor | None = None,
                          stream=None) -> torch.Tensor:
    """Psi_r(g) from the all-reduced limbs of psi_r_shard_g (device float64[1])."""
    with _On(total.device, stream) as on:
        out = torch.empty(1, dtype=torch.float64, device=total.device) if out is None else out
        _check(lib().plugin_psi_from_total(total.data_ptr(), int(n), float(g), int(r), out.data_ptr(), on.handle))
    return out


def plugin_after_psi6(total: torch.Tensor, out: torch.Tensor, stream=None):
    with _On(out.device, stream) as on:
        _check(lib().plugin_after_psi6(total.data_ptr(), out.data_ptr(), on.handle))
    return out


def plugin_after_psi4(total: torch.Tensor, out: torch.Tensor, stream=None):
    with _On(out.device, stream) as on:
        _check(lib().plugin_after_psi4(total.data_ptr(), out.data_ptr(), on.handle))
    return out


def plugin_num_tiles(n: int, r: int) -> int:
    """Work items of the order-r pass for n samples (tiles; a function of n and r)."""
    return lib().plugin_num_tiles(n, r)


def plugin_tile_edge(n: int, r: int) -> int:
    return lib().plugin_tile_edge(n, r)


def plugin_work_item(n: int, r: int, item: int) -> tuple[tuple[int, int], tuple[int, int], int]:
    """The pairs of work item `item` of the order-r pass: (row range, column range, weight)."""
    out = (ctypes.c_int64 * 5)()
    if lib().plugin_work_item(n, r, item, out) != 0:
        raise IndexError(f"work item {item} out of range for n={n}")
    return (out[0], out[1]), (out[2], out[3]), out[4]


def plugin_shard_tiles(n: int, r: int, rank: int, world: int) -> tuple[int, int]:
    b, e = ctypes.c_int64(), ctypes.c_int64()
    lib().plugin_shard_tiles(n, r, rank, world, ctypes.byref(b), ctypes.byref(e))
    return b.value, e.value


DPI_RESULT_BYTES = ctypes.sizeof(plugin_dpi_result)


def plugin_dpi(x: torch.Tensor, stages: int, out: torch.Tensor | None = None, ws: torch.Tensor | None = None,
               stream=None) -> torch.Tensor:
    """l-stage direct plug-in (Alg. 1 is stages = 2) on the device; returns the result buffer."""
    with _On(_dev(x), stream) as on:
        x = _x(x)
        on.uses(x)
        n = x.numel()
        ws = workspace(n, x.device) if ws is None else ws
        out = torch.empty(DPI_RESULT_BYTES, dtype=torch.uint8, device=x.device) if out is None else out
        _check(lib().plugin_dpi(x.data_ptr(), n, int(stages), out.data_ptr(), ws.data_ptr(), ws.numel(), on.handle))
    return out


def read_dpi_result(buf: torch.Tensor) -> dict:
    return plugin_dpi_result.from_buffer_copy(buf.detach().to("cpu").numpy().tobytes()).to_dict()


def psi_r_q32(zq: torch.Tensor, rg_q: int, r: int, ws: torch.Tensor | None = None, stream=None) -> int:
    """sum_i sum_j term(zq_i - zq_j) in Q32.32 (NEXT 2) as an exact Python int (synchronises)."""
    if not (isinstance(zq, torch.Tensor) and zq.is_cuda and zq.dtype == torch.int64 and zq.dim() == 1):
        raise TypeError("zq must be a 1-D CUDA int64 tensor (Q32.32 raw values)")
    with _On(zq.device, stream) as on:
        zq = zq.contiguous()
        on.uses(zq)
        n = zq.numel()
        ws = workspace(n, zq.device) if ws is None else ws
        out = torch.zeros(2, dtype=torch.int64, device=zq.device)
        _check(lib().psi_r_q32(zq.data_ptr(), n, int(rg_q), int(r), out.data_ptr(), ws.data_ptr(), ws.numel(),
                               on.handle))
        lo, hi = out.cpu().tolist()
    return hi * (1 << 64) + (lo & ((1 << 64) - 1))


def plugin_h_q32(x: torch.Tensor, out: torch.Tensor | None = None, ws: torch.Tensor | None = None, stream=None):
    """Alg. 1 with the Q32.32 pair passes (asynchronous); returns the device result buffer."""
    with _On(_dev(x), stream) as on:
        x = _x(x)
        on.uses(x)
        n = x.numel()
        if ws is None:
            nbytes = lib().plugin_q32_workspace_bytes(n)
            t = torch.empty(nbytes + 256, dtype=torch.uint8, device=x.device)
            off = (-t.data_ptr()) % 256
            ws = t[off:off + nbytes]
        out = new_result(x.device) if out is None else out
        _check(lib().plugin_h_q32(x.data_ptr(), n, out.data_ptr(), ws.data_ptr(), ws.numel(), on.handle))
    return out


def kde_workspace_bytes(n: int, m: int) -> int:
    return lib().kde_workspace_bytes(n, m)


def kde_workspace(n: int, m: int, device=None) -> torch.Tensor:
    nbytes = kde_workspace_bytes(n, m)
    t = torch.empty(nbytes + 256, dtype=torch.uint8, device=device or "cuda")
    off = (-t.data_ptr()) % 256
    return t[off:off + nbytes]


def kde_eval(x: torch.Tensor, h: float, points: torch.Tensor, out: torch.Tensor | None = None,
             ws: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """f(x_k, h) of Eq. 1-2 at every point (device float64[m], asynchronous)."""
    with _On(_dev(x), stream) as on:
        x = _x(x)
        on.uses(x)
        points = _x(points)
        on.uses(points)
        n, m = x.numel(), points.numel()
        ws = kde_workspace(n, m, x.device) if ws is None else ws
        out = torch.empty(m, dtype=torch.float64, device=x.device) if out is None else out
        _check(lib().kde_eval(x.data_ptr(), n, float(h), points.data_ptr(), m, out.data_ptr(), ws.data_ptr(),
                              ws.numel(), on.handle))
    return out


def kde_prepare(x: torch.Tensor, ws: torch.Tensor, stream=None) -> torch.Tensor:
    """Sort X into the KDE workspace once (then kde_eval_prepared for any points / h)."""
    with _On(_dev(x), stream) as on:
        x = _x(x)
        on.uses(x)
        _check(lib().kde_prepare(x.data_ptr(), x.numel(), ws.data_ptr(), ws.numel(), on.handle))
    return ws


def kde_eval_prepared(n: int, h: float, points: torch.Tensor, ws: torch.Tensor, out: torch.Tensor | None = None,
                      stream=None) -> torch.Tensor:
    with _On(_dev(points), stream) as on:
        points = _x(points)
        on.uses(points, ws)
        m = points.numel()
        out = torch.empty(m, dtype=torch.float64, device=points.device) if out is None else out
        _check(lib().kde_eval_prepared(int(n), float(h), points.data_ptr(), m, out.data_ptr(), ws.data_ptr(),
                                       ws.numel(), on.handle))
    return out


def plugin_sort(x: torch.Tensor, ws: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """The sorted copy of X the passes read (device float32, asynchronous)."""
    with _On(_dev(x), stream) as on:
        x = _x(x)
        on.uses(x)
        n = x.numel()
        ws = workspace(n, x.device) if ws is None else ws
        out = torch.empty_like(x)
        _check(lib().plugin_sort(x.data_ptr(), n, out.data_ptr(), ws.data_ptr(), ws.numel(), on.handle))
    return out


def plugin_last_error() -> str:
    return lib().plugin_last_error().decode()


def plugin_version() -> str:
    return lib().plugin_version().decode()
