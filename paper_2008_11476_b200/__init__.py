"""graphvx-b200: B200-native execution backend for the OpenVX graph path of
HipaccVX (arXiv:2008.11476).

The product is native code: the C++ graph API (``include/graphvx``, in
``lib/libgraphvx.so``) over the sm_100a device runtime (``include/gvxb.h``,
``lib/libgvx_cuda.so``).  This module only loads those libraries with
ctypes and mirrors the C facade (``include/gvx_c.h``) for Python hosts
(tests, ``bench.py``).  There is no Python or host compute path: on a
machine without a CUDA device every execution call raises ``GraphvxError``.
"""
from __future__ import annotations

import ctypes
import os
import pathlib
import subprocess

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
REPO = ROOT.parent
LIB_DIR = ROOT / "lib"
LIB_CUDA = LIB_DIR / "libgvx_cuda.so"
LIB_GRAPH = LIB_DIR / "libgraphvx.so"

# gvx::ErrorCode names, index = status - 1 (include/graphvx/error.hpp)
ERROR_CODES = [
    "ZeroDimension", "BadFormat", "BadKernel", "AccessDenied", "UnknownObject", "UnknownKernel",
    "CrossGraphVirtual", "MultipleWriters", "CycleDetected", "UnstampedGraph", "MissingInput",
    "ShapeMismatch", "DivByZero", "TypeMismatch", "MissingCast", "OffsetOutOfWindow", "UnsupportedKind",
    "NonStreamable", "IoError", "SchemaError",
]

# exact output formats of the five configurations
CONFIG_OUTPUT = {1: np.int16, 2: np.uint8, 3: np.uint8, 4: None, 5: np.int16}
CONFIG_SEED = {1: 1, 2: 2, 3: 3, 4: 4, 5: 5}
CONFIG_SIZE = {1: (1920, 1080), 2: (3840, 2160), 3: (7680, 4320), 4: (3840, 2160), 5: (16384, 16384)}
CONFIG_FRAMES = {1: 1, 2: 1, 3: 1, 4: 64, 5: 1}


class GraphvxError(RuntimeError):
    def __init__(self, status: int, message: str):
        name = ERROR_CODES[status - 1] if 1 <= status <= len(ERROR_CODES) else f"status{status}"
        super().__init__(f"{name}: {message}")
        self.status = status
        self.code = name


def build(verbose: bool = False) -> None:
    """Compile the native libraries in-tree (make)."""
    out = subprocess.run(["make", "-j8", "-C", str(REPO)], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("native build failed:\n" + out.stdout[-4000:] + out.stderr[-4000:])
    if verbose:
        print(out.stdout[-2000:])


_cuda = None
_graph = None


def _load():
    global _cuda, _graph
    if _graph is not None:
        return _cuda, _graph
    if not LIB_GRAPH.exists() or not LIB_CUDA.exists():
        raise ImportError(f"graphvx-b200 native libraries missing in {LIB_DIR}; run build()")
    _cuda = ctypes.CDLL(str(LIB_CUDA), mode=ctypes.RTLD_GLOBAL)
    _graph = ctypes.CDLL(str(LIB_GRAPH), mode=ctypes.RTLD_GLOBAL)
    _declare(_cuda, _graph)
    return _cuda, _graph


def _declare(c, g):
    P, I, L, D, U8P = ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_double, ctypes.c_void_p
    c.gvxb_last_error.restype = ctypes.c_char_p
    c.gvxb_device_count.argtypes = [ctypes.POINTER(I)]
    c.gvxb_ctx_create.argtypes = [I, ctypes.POINTER(P)]
    c.gvxb_ctx_destroy.argtypes = [P]
    c.gvxb_ctx_stream.argtypes = [P]
    c.gvxb_ctx_stream.restype = P
    c.gvxb_ctx_set_stream.argtypes = [P, P]
    c.gvxb_sync.argtypes = [P]
    c.gvxb_alloc.argtypes = [P, ctypes.c_size_t, ctypes.POINTER(P)]
    c.gvxb_free.argtypes = [P, P]
    c.gvxb_host_alloc.argtypes = [ctypes.c_size_t, ctypes.POINTER(P)]
    c.gvxb_host_free.argtypes = [P]
    c.gvxb_memset.argtypes = [P, P, I, ctypes.c_size_t]
    c.gvxb_upload_2d.argtypes = [P, P, ctypes.c_size_t, P, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_size_t]
    c.gvxb_download_2d.argtypes = [P, P, ctypes.c_size_t, P, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_size_t]
    c.gvxb_event_create.argtypes = [ctypes.POINTER(P)]
    c.gvxb_event_destroy.argtypes = [P]
    c.gvxb_event_record.argtypes = [P, P]
    c.gvxb_event_elapsed_ms.argtypes = [P, P, ctypes.POINTER(ctypes.c_float)]
    c.gvxb_launch_count.argtypes = [P]
    c.gvxb_launch_count.restype = ctypes.c_int64
    c.gvxb_band_rows.argtypes = [ctypes.c_int32] * 3 + [ctypes.POINTER(ctypes.c_int32)] * 2
    g.gvxc_last_error.restype = ctypes.c_char_p
    g.gvxc_config_create.argtypes = [I, I, I, I, ctypes.POINTER(P)]
    g.gvxc_graph_destroy.argtypes = [P]
    g.gvxc_graph_describe.argtypes = [P, I, ctypes.c_char_p, ctypes.c_size_t]
    g.gvxc_graph_pass_stats.argtypes = [P, ctypes.POINTER(L)]
    g.gvxc_graph_run_host.argtypes = [P, I, U8P, P, ctypes.POINTER(L), ctypes.POINTER(D), ctypes.POINTER(L)]
    g.gvxc_session_create.argtypes = [P, I, I, ctypes.POINTER(P)]
    g.gvxc_session_destroy.argtypes = [P]
    g.gvxc_session_bind.argtypes = [P, I, P, ctypes.c_int64, ctypes.c_int64]
    g.gvxc_session_set_stream.argtypes = [P, P]
    g.gvxc_session_launch.argtypes = [P]
    g.gvxc_session_set_overlap.argtypes = [P, I]
    g.gvxc_session_sync.argtypes = [P]
    g.gvxc_session_launches.argtypes = [P]
    g.gvxc_session_upload_input.argtypes = [P, I, U8P]
    g.gvxc_session_download.argtypes = [P, I, I, P, ctypes.POINTER(L), ctypes.POINTER(D)]
    g.gvxc_random_u8.argtypes = [I, I, ctypes.c_ulonglong, U8P]
    g.gvxc_pipeline_create.argtypes = [P, I, I, ctypes.POINTER(P)]
    g.gvxc_pipeline_destroy.argtypes = [P]
    g.gvxc_pipeline_submit.argtypes = [P, U8P]
    g.gvxc_pipeline_submit_pinned.argtypes = [P, U8P]
    g.gvxc_host_register.argtypes = [P, ctypes.c_size_t]
    g.gvxc_host_unregister.argtypes = [P]
    g.gvxc_pipeline_pending.argtypes = [P]
    g.gvxc_pipeline_next.argtypes = [P, P, ctypes.POINTER(L), ctypes.POINTER(D), ctypes.POINTER(L)]
    g.gvxc_pipeline_next_view.argtypes = [P, ctypes.POINTER(P), ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(L)]
    g.gvxc_pipeline_stream.argtypes = [P, ctypes.POINTER(P), I, I, P, P, ctypes.POINTER(L)]
    g.gvxc_graph_input_ptr.argtypes = [P, ctypes.POINTER(P), ctypes.POINTER(ctypes.c_size_t)]
    g.gvxc_graph_output_ptr.argtypes = [P, ctypes.POINTER(P), ctypes.POINTER(ctypes.c_size_t)]
    g.gvxc_launch_count.restype = ctypes.c_longlong
    g.gvxc_default_stream.restype = P
    SZ = ctypes.c_size_t
    g.gvxc_json_roundtrip.argtypes = [ctypes.c_char_p, ctypes.c_char_p, SZ, ctypes.POINTER(SZ)]
    g.gvxc_json_load.argtypes = [ctypes.c_char_p, ctypes.POINTER(P)]
    g.gvxc_json_destroy.argtypes = [P]
    g.gvxc_json_run.argtypes = [P, I, ctypes.c_ulonglong, U8P, SZ, ctypes.POINTER(SZ), ctypes.POINTER(L)]
    g.gvxc_json_pass_stats.argtypes = [P, ctypes.POINTER(L)]
    g.gvxc_json_describe.argtypes = [P, I, ctypes.c_char_p, ctypes.c_size_t]
    g.gvxc_json_bench.argtypes = [P, I, I, I, ctypes.c_ulonglong, ctypes.POINTER(D)]
    I32P = ctypes.POINTER(ctypes.c_int32)
    c.gvxb_band_plan_make.argtypes = [ctypes.c_int32] * 4 + [ctypes.c_void_p]
    c.gvxb_comm_available.restype = I
    c.gvxb_comm_unique_id.argtypes = [ctypes.c_void_p]
    c.gvxb_comm_create.argtypes = [I, I, I, ctypes.c_void_p, ctypes.POINTER(P)]
    c.gvxb_comm_destroy.argtypes = [P]
    c.gvxb_comm_allreduce_max.argtypes = [P, ctypes.POINTER(D)]
    c.gvxb_comm_barrier.argtypes = [P]
    g.gvxc_band_create.argtypes = [P, I, I, P, I, I, ctypes.POINTER(P)]
    g.gvxc_band_destroy.argtypes = [P]
    g.gvxc_band_layout.argtypes = [P, I32P]
    g.gvxc_band_tensor.argtypes = [P, I, ctypes.POINTER(P), ctypes.POINTER(ctypes.c_int64),
                                   ctypes.POINTER(ctypes.c_int64), I32P, I32P]
    g.gvxc_band_upload.argtypes = [P, I, P, SZ, I, I, I]
    g.gvxc_band_download.argtypes = [P, I, P, SZ, I, I, I]
    g.gvxc_band_set_stream.argtypes = [P, P]
    g.gvxc_band_set_overlap.argtypes = [P, I]
    g.gvxc_band_bind.argtypes = [P, I, P, ctypes.c_int64, ctypes.c_int64]
    g.gvxc_band_launch.argtypes = [P]
    g.gvxc_band_sync.argtypes = [P]
    g.gvxc_band_launches.argtypes = [P]
    g.gvxc_band_run_host.argtypes = [P, P, SZ, I, P, SZ, I]
    g.gvxc_band_describe.argtypes = [P, ctypes.c_char_p, SZ]
    g.gvxc_group_create.argtypes = [P, I, ctypes.POINTER(I), I, ctypes.POINTER(P)]
    g.gvxc_group_destroy.argtypes = [P]
    g.gvxc_group_band.argtypes = [P, I, ctypes.POINTER(P)]
    g.gvxc_group_launch.argtypes = [P]
    g.gvxc_group_sync.argtypes = [P]


def _check_graph(rc: int):
    if rc != 0:
        raise GraphvxError(rc, _graph.gvxc_last_error().decode(errors="replace"))


def _check_cuda(rc: int):
    if rc != 0:
        raise GraphvxError(rc, _cuda.gvxb_last_error().decode(errors="replace"))


def libraries():
    return _load()


def device_count() -> int:
    c, _ = _load()
    n = ctypes.c_int(0)
    c.gvxb_device_count(ctypes.byref(n))
    return n.value


def launch_count() -> int:
    """Device kernels launched so far by the library's context (-1: no device)."""
    _, g = _load()
    return int(g.gvxc_launch_count())


def random_u8(width: int, height: int, seed: int) -> np.ndarray:
    """Reference-identical synthetic U8 image (random_buffer, mt19937_64)."""
    _, g = _load()
    out = np.empty((height, width), np.uint8)
    _check_graph(g.gvxc_random_u8(width, height, seed, out.ctypes.data))
    return out


def parse_outputs(blob: bytes):
    """Declared outputs serialised by configs/json_runner.hpp:
    [u32 kind][u32 n][payload]...; returns [(kind, bytes)]."""
    out, i = [], 0
    while i < len(blob):
        kind = int.from_bytes(blob[i:i + 4], "little")
        n = int.from_bytes(blob[i + 4:i + 8], "little")
        out.append((kind, bytes(blob[i + 8:i + 8 + n])))
        i += 8 + n
    return out


def json_roundtrip(text: str) -> str:
    """save_graph_json(load_graph_json(text)) (graph_io.hpp)."""
    _, g = _load()
    need = ctypes.c_size_t()
    _check_graph(g.gvxc_json_roundtrip(text.encode(), None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    _check_graph(g.gvxc_json_roundtrip(text.encode(), buf, need.value, ctypes.byref(need)))
    return buf.value.decode()


class GraphFile:
    """A graph-description file loaded through graph_io + verify/expand/
    optimize; run() executes run_plan / run_naive on random_buffer inputs."""

    def __init__(self, text: str):
        _, self._g = _load()
        self._h = ctypes.c_void_p()
        _check_graph(self._g.gvxc_json_load(text.encode(), ctypes.byref(self._h)))

    def __del__(self):
        if getattr(self, "_h", None):
            self._g.gvxc_json_destroy(self._h)
            self._h = None

    def run(self, naive: bool = False, seed: int = 1):
        need = ctypes.c_size_t()
        counters = (ctypes.c_longlong * 4)()
        _check_graph(self._g.gvxc_json_run(self._h, int(naive), seed, None, 0, ctypes.byref(need), counters))
        buf = (ctypes.c_uint8 * max(1, need.value))()
        _check_graph(self._g.gvxc_json_run(self._h, int(naive), seed, buf, need.value, ctypes.byref(need), counters))
        names = ["kernel_launches", "pixels_read", "pixels_written", "transfers_executed"]
        return parse_outputs(bytes(buf)[:need.value]), dict(zip(names, list(counters)))

    def describe(self, naive: bool = False) -> str:
        buf = ctypes.create_string_buffer(8192)
        _check_graph(self._g.gvxc_json_describe(self._h, int(naive), buf, 8192))
        return buf.value.decode()

    def bench(self, naive: bool = False, frames: int = 1, iters: int = 20, seed: int = 1) -> dict:
        """Device time of one execution over `frames` frames (DeviceSession)."""
        out = (ctypes.c_double * 4)()
        _check_graph(self._g.gvxc_json_bench(self._h, int(naive), frames, iters, seed, out))
        return {"ms": out[0], "bytes": out[1], "launches": out[2], "frames": int(out[3])}

    def pass_stats(self) -> dict:
        st = (ctypes.c_longlong * 8)()
        _check_graph(self._g.gvxc_json_pass_stats(self._h, st))
        keys = ["nodes_before", "nodes_alive", "nodes_removed", "transfers_naive", "transfers_optimized",
                "fused_groups", "launches_before", "launches_after"]
        return dict(zip(keys, list(st)))


class ConfigGraph:
    """One BASELINE configuration built through the public API (verify ->
    expand -> verify -> optimize)."""

    def __init__(self, cfg: int, width: int, height: int, virtual_mid: bool = True):
        _, g = _load()
        self.cfg, self.width, self.height = cfg, width, height
        h = ctypes.c_void_p()
        _check_graph(g.gvxc_config_create(cfg, width, height, int(virtual_mid), ctypes.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            _graph.gvxc_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def describe(self, naive: bool = False) -> str:
        buf = ctypes.create_string_buffer(8192)
        _check_graph(_graph.gvxc_graph_describe(self._h, int(naive), buf, len(buf)))
        return buf.value.decode()

    def pass_stats(self) -> dict:
        st = (ctypes.c_longlong * 8)()
        _graph.gvxc_graph_pass_stats(self._h, st)
        keys = ["nodes_before", "nodes_alive", "nodes_removed", "transfers_naive", "transfers_optimized",
                "fused_groups", "launches_before", "launches_after"]
        return dict(zip(keys, list(st)))

    def output_array(self):
        dt = CONFIG_OUTPUT[self.cfg]
        return None if dt is None else np.empty((self.height, self.width), dt)

    def run_host(self, image: np.ndarray, naive: bool = False, out: np.ndarray | None = None):
        """run_plan / run_naive with host buffers.  Returns (result, counters)
        where result is the output plane (written into `out` when given: a
        caller reusing one destination array across frames), or (hist, mean,
        stddev) for cfg4."""
        img = np.ascontiguousarray(image, dtype=np.uint8)
        assert img.shape == (self.height, self.width)
        if out is None:
            out = self.output_array()
        else:
            assert out.shape == (self.height, self.width) and out.dtype == np.dtype(CONFIG_OUTPUT[self.cfg])
            assert out.flags.c_contiguous
        hist = (ctypes.c_longlong * 256)()
        stats = (ctypes.c_double * 2)()
        counters = (ctypes.c_longlong * 4)()
        _check_graph(_graph.gvxc_graph_run_host(self._h, int(naive), img.ctypes.data,
                                                None if out is None else out.ctypes.data, hist, stats, counters))
        cnt = dict(zip(["kernel_launches", "pixels_read", "pixels_written", "transfers_executed"], list(counters)))
        if self.cfg == 4:
            return (np.array(list(hist), np.int64), stats[0], stats[1]), cnt
        return out, cnt

    def run_host_inplace(self, image: np.ndarray, naive: bool = False):
        """run_plan / run_naive with host buffers, leaving the result in the
        graph's own (page-locked) output buffer instead of copying it out:
        returns (read-only view of the output plane or cfg4 stats, counters).
        The view is valid until the next host run."""
        img = np.ascontiguousarray(image, dtype=np.uint8)
        hist = (ctypes.c_longlong * 256)()
        stats = (ctypes.c_double * 2)()
        counters = (ctypes.c_longlong * 4)()
        _check_graph(_graph.gvxc_graph_run_host(self._h, int(naive), img.ctypes.data, None, hist, stats, counters))
        cnt = dict(zip(["kernel_launches", "pixels_read", "pixels_written", "transfers_executed"], list(counters)))
        if self.cfg == 4:
            return (np.array(list(hist), np.int64), stats[0], stats[1]), cnt
        ptr, n = ctypes.c_void_p(), ctypes.c_size_t()
        _check_graph(_graph.gvxc_graph_output_ptr(self._h, ctypes.byref(ptr), ctypes.byref(n)))
        dt = np.dtype(CONFIG_OUTPUT[self.cfg])
        view = np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctypes.c_uint8)), shape=(n.value,))
        return view.view(dt).reshape(self.height, self.width), cnt


class Pipeline:
    """gvx::HostPipeline over a ConfigGraph: submit host frames, get results
    back in order, with up to `depth` frames in flight."""

    def __init__(self, graph: "ConfigGraph", depth: int = 3, naive: bool = False):
        self.graph = graph
        self._h = ctypes.c_void_p()
        _check_graph(_graph.gvxc_pipeline_create(graph._h, int(naive), depth, ctypes.byref(self._h)))

    def __del__(self):
        if getattr(self, "_h", None):
            _graph.gvxc_pipeline_destroy(self._h)
            self._h = None

    def submit(self, image: np.ndarray, pinned: bool = False):
        """Copies the frame into the pipeline's page-locked staging, or with
        `pinned` DMAs it straight from `image` (which must be page-locked,
        see PinnedHost, and stay unchanged until its result is taken)."""
        img = np.ascontiguousarray(image, dtype=np.uint8)
        assert img.shape == (self.graph.height, self.graph.width)
        if pinned:
            assert img.ctypes.data == image.ctypes.data, "a pinned frame must be a contiguous uint8 array"
            _check_graph(_graph.gvxc_pipeline_submit_pinned(self._h, img.ctypes.data))
        else:
            _check_graph(_graph.gvxc_pipeline_submit(self._h, img.ctypes.data))

    def pending(self) -> int:
        return _graph.gvxc_pipeline_pending(self._h)

    def next_view(self):
        """Oldest frame's output plane as a read-only view of the pipeline's
        page-locked staging (valid until the next submit), and counters."""
        ptr, n = ctypes.c_void_p(), ctypes.c_size_t()
        counters = (ctypes.c_longlong * 4)()
        _check_graph(_graph.gvxc_pipeline_next_view(self._h, ctypes.byref(ptr), ctypes.byref(n), counters))
        views = self.__dict__.setdefault("_views", {})  # one numpy view per staging buffer
        key = (ptr.value, n.value)
        if key not in views:
            dt = np.dtype(CONFIG_OUTPUT[self.graph.cfg])
            raw = np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctypes.c_uint8)), shape=(n.value,))
            views[key] = raw.view(dt).reshape(self.graph.height, self.graph.width)
        cnt = dict(zip(["kernel_launches", "pixels_read", "pixels_written", "transfers_executed"], list(counters)))
        return views[key], cnt

    _ON_RESULT = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)

    def stream(self, frames, pinned: bool = False, on_result=None) -> dict:
        """All `frames` through the pipeline in one native call (results are
        taken in order from page-locked staging, `depth` frames in flight);
        returns the summed counters.  `on_result(view)` (optional) sees each
        result plane while it is valid.  With `pinned` every frame must be
        page-locked (PinnedHost)."""
        ptrs = (ctypes.c_void_p * len(frames))()
        for i, f in enumerate(frames):
            assert f.dtype == np.uint8 and f.flags.c_contiguous and f.shape == (self.graph.height, self.graph.width)
            ptrs[i] = f.ctypes.data
        cb = None
        if on_result is not None:
            dt = np.dtype(CONFIG_OUTPUT[self.graph.cfg])

            def _cb(view, nbytes, _user):
                raw = np.ctypeslib.as_array(ctypes.cast(view, ctypes.POINTER(ctypes.c_uint8)), shape=(nbytes,))
                on_result(raw.view(dt).reshape(self.graph.height, self.graph.width))

            cb = self._ON_RESULT(_cb)
        counters = (ctypes.c_longlong * 4)()
        _check_graph(_graph.gvxc_pipeline_stream(self._h, ctypes.cast(ptrs, ctypes.POINTER(ctypes.c_void_p)),
                                                 len(frames), int(pinned), ctypes.cast(cb, ctypes.c_void_p) if cb
                                                 else None, None, counters))
        return dict(zip(["kernel_launches", "pixels_read", "pixels_written", "transfers_executed"], list(counters)))

    def next(self, out: np.ndarray = None):
        """Oldest frame's result: (output plane, counters), or
        ((hist, mean, stddev), counters) for config 4."""
        if out is None:
            out = self.graph.output_array()
        hist = (ctypes.c_longlong * 256)()
        stats = (ctypes.c_double * 2)()
        counters = (ctypes.c_longlong * 4)()
        _check_graph(_graph.gvxc_pipeline_next(self._h, None if out is None else out.ctypes.data, hist, stats, counters))
        cnt = dict(zip(["kernel_launches", "pixels_read", "pixels_written", "transfers_executed"], list(counters)))
        if self.graph.cfg == 4:
            return (np.array(list(hist), np.int64), stats[0], stats[1]), cnt
        return out, cnt


class PinnedHost:
    """Page-locks (cudaHostRegister) the memory of host arrays for the
    lifetime of the object, so Pipeline.submit(..., pinned=True) DMAs from
    them directly; releases them on close()."""

    def __init__(self, arrays):
        _load()
        self._ptrs = []
        try:
            for a in arrays:
                assert a.flags["C_CONTIGUOUS"]
                _check_graph(_graph.gvxc_host_register(a.ctypes.data, a.nbytes))
                self._ptrs.append(a.ctypes.data)
        except BaseException:
            self.close()
            raise

    def close(self):
        for p in self._ptrs:
            _graph.gvxc_host_unregister(p)
        self._ptrs = []

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        if getattr(self, "_ptrs", None):
            self.close()


class Session:
    """Device-resident execution of a ConfigGraph over `frames` frames."""

    def __init__(self, graph: ConfigGraph, frames: int = 1, naive: bool = False):
        self.graph, self.frames = graph, frames
        h = ctypes.c_void_p()
        _check_graph(_graph.gvxc_session_create(graph.handle, int(naive), frames, ctypes.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            _graph.gvxc_session_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def bind(self, slot: int, dptr: int, pitch: int, frame_stride: int = 0):
        _check_graph(_graph.gvxc_session_bind(self._h, slot, ctypes.c_void_p(dptr), pitch, frame_stride))

    def set_stream(self, stream: int | None):
        _check_graph(_graph.gvxc_session_set_stream(self._h, ctypes.c_void_p(stream or 0)))

    def set_overlap(self, mode: int):
        _check_graph(_graph.gvxc_session_set_overlap(self._h, mode))

    def launch(self):
        _check_graph(_graph.gvxc_session_launch(self._h))

    def sync(self):
        _check_graph(_graph.gvxc_session_sync(self._h))

    def launches(self) -> int:
        return _graph.gvxc_session_launches(self._h)

    def upload(self, frame: int, image: np.ndarray):
        img = np.ascontiguousarray(image, dtype=np.uint8)
        _check_graph(_graph.gvxc_session_upload_input(self._h, frame, img.ctypes.data))

    def download(self, frame: int = 0, slot: int = 1):
        out = self.graph.output_array()
        hist = (ctypes.c_longlong * 256)()
        stats = (ctypes.c_double * 2)()
        _check_graph(_graph.gvxc_session_download(self._h, slot, frame, None if out is None else out.ctypes.data,
                                                  hist, stats))
        if self.graph.cfg == 4:
            return np.array(list(hist), np.int64), stats[0], stats[1]
        return out


class Device:
    """Thin wrapper over a gvxb context (device memory, events, stream)."""

    def __init__(self, device: int = 0):
        c, _ = _load()
        self.c = c
        h = ctypes.c_void_p()
        _check_cuda(c.gvxb_ctx_create(device, ctypes.byref(h)))
        self.h = h

    @property
    def stream(self) -> int:
        return self.c.gvxb_ctx_stream(self.h) or 0

    def alloc(self, nbytes: int) -> int:
        p = ctypes.c_void_p()
        _check_cuda(self.c.gvxb_alloc(self.h, nbytes, ctypes.byref(p)))
        return p.value

    def free(self, ptr: int):
        self.c.gvxb_free(self.h, ctypes.c_void_p(ptr))

    def upload(self, dptr: int, dpitch: int, arr: np.ndarray):
        a = np.ascontiguousarray(arr)
        row = a.shape[-1] * a.itemsize
        rows = a.size * a.itemsize // row
        _check_cuda(self.c.gvxb_upload_2d(self.h, ctypes.c_void_p(dptr), dpitch, a.ctypes.data, row, row, rows))

    def download(self, arr: np.ndarray, dptr: int, dpitch: int):
        row = arr.shape[-1] * arr.itemsize
        rows = arr.size * arr.itemsize // row
        _check_cuda(self.c.gvxb_download_2d(self.h, arr.ctypes.data, row, ctypes.c_void_p(dptr), dpitch, row, rows))
        self.sync()

    def memset(self, dptr: int, value: int, nbytes: int):
        _check_cuda(self.c.gvxb_memset(self.h, ctypes.c_void_p(dptr), value, nbytes))

    def sync(self):
        _check_cuda(self.c.gvxb_sync(self.h))

    def event(self) -> int:
        e = ctypes.c_void_p()
        _check_cuda(self.c.gvxb_event_create(ctypes.byref(e)))
        return e.value

    def record(self, ev: int):
        _check_cuda(self.c.gvxb_event_record(self.h, ctypes.c_void_p(ev)))

    def elapsed_ms(self, a: int, b: int) -> float:
        ms = ctypes.c_float()
        _check_cuda(self.c.gvxb_event_elapsed_ms(ctypes.c_void_p(a), ctypes.c_void_p(b), ctypes.byref(ms)))
        return ms.value

    def launch_count(self) -> int:
        return int(self.c.gvxb_launch_count(self.h))


class GvxbImage(ctypes.Structure):
    """include/gvxb.h gvxb_image."""
    _fields_ = [("data", ctypes.c_void_p), ("pitch", ctypes.c_int64), ("width", ctypes.c_int32),
                ("height", ctypes.c_int32), ("format", ctypes.c_int32), ("frames", ctypes.c_int32),
                ("frame_stride", ctypes.c_int64)]


class GvxbBand(ctypes.Structure):
    """include/gvxb.h gvxb_band."""
    _fields_ = [("row0", ctypes.c_int32), ("row1", ctypes.c_int32), ("global_h", ctypes.c_int32),
                ("src_row0", ctypes.c_int32), ("dst_row0", ctypes.c_int32)]


class GvxbEdgeArgs(ctypes.Structure):
    """include/gvxb.h gvxb_edge_args."""
    _fields_ = [("src", GvxbImage), ("gx", GvxbImage), ("gy", GvxbImage), ("mag", GvxbImage),
                ("with_gauss", ctypes.c_int32), ("band", GvxbBand)]


def edge_band(device: "Device", src_ptr: int, src_pitch: int, width: int, src_rows: int, mag_ptr: int,
              mag_pitch: int, row0: int, row1: int, global_h: int, src_row0: int, dst_row0: int,
              with_gauss: bool = True):
    """Fused Gaussian3x3 -> Sobel3x3 -> Magnitude on global rows [row0, row1)
    of a row band (gvxb_edge); `src` holds global rows from src_row0."""
    c, _ = _load()
    c.gvxb_edge.argtypes = [ctypes.c_void_p, ctypes.POINTER(GvxbEdgeArgs)]
    a = GvxbEdgeArgs()
    a.src = GvxbImage(src_ptr, src_pitch, width, src_rows, 0, 1, 0)
    a.mag = GvxbImage(mag_ptr, mag_pitch, width, row1 - row0, 2, 1, 0)
    a.with_gauss = int(with_gauss)
    a.band = GvxbBand(row0, row1, global_h, src_row0, dst_row0)
    _check_cuda(c.gvxb_edge(device.h, ctypes.byref(a)))


class GvxbStencilArgs(ctypes.Structure):
    """include/gvxb.h gvxb_stencil_args."""
    _fields_ = [("src", GvxbImage), ("dst", GvxbImage), ("ksize", ctypes.c_int32),
                ("mask", ctypes.c_int32 * 49), ("div_num", ctypes.c_int64), ("div_den", ctypes.c_int64),
                ("mode", ctypes.c_int32), ("band", GvxbBand)]


class GvxbConvStatsArgs(ctypes.Structure):
    """include/gvxb.h gvxb_conv_stats_args."""
    _fields_ = [("src", GvxbImage), ("converted", GvxbImage), ("ksize", ctypes.c_int32),
                ("mask", ctypes.c_int32 * 49), ("scale", ctypes.c_int64), ("conv_format", ctypes.c_int32),
                ("shift", ctypes.c_int32), ("wrap", ctypes.c_int32), ("bins", ctypes.c_int32),
                ("offset", ctypes.c_int64), ("range", ctypes.c_int64), ("hist", ctypes.c_void_p),
                ("sum", ctypes.c_void_p), ("sumsq", ctypes.c_void_p), ("mean", ctypes.c_void_p),
                ("stddev", ctypes.c_void_p), ("work", ctypes.c_void_p)]


def _mask49(mask):
    m = (ctypes.c_int32 * 49)()
    for i, v in enumerate(np.asarray(mask, np.int64).ravel()):
        m[i] = int(v)
    return m


class GvxbHarrisArgs(ctypes.Structure):
    """include/gvxb.h gvxb_harris_args."""
    _fields_ = [("src", GvxbImage), ("mask", GvxbImage), ("response", GvxbImage), ("k", ctypes.c_double),
                ("threshold", ctypes.c_double), ("band", GvxbBand)]


def harris(device: "Device", img: np.ndarray, k: float, threshold: float, response: bool = False):
    """Host wrapper over gvxb_harris on one U8 frame: returns the U8 mask
    (and the F32 response image when `response`)."""
    c, _ = _load()
    c.gvxb_harris.argtypes = [ctypes.c_void_p, ctypes.POINTER(GvxbHarrisArgs)]
    h, w = img.shape
    pitch = (w + 127) // 128 * 128
    src, dst = device.alloc(pitch * h), device.alloc(pitch * h)
    rsp = device.alloc(4 * pitch * h) if response else 0
    try:
        device.upload(src, pitch, np.ascontiguousarray(img, np.uint8))
        a = GvxbHarrisArgs()
        a.src = GvxbImage(src, pitch, w, h, 0, 1, 0)
        a.mask = GvxbImage(dst, pitch, w, h, 0, 1, 0)
        a.response = GvxbImage(rsp or None, 4 * pitch, w, h, 4, 1, 0)
        a.k, a.threshold = float(k), float(threshold)
        a.band = GvxbBand(0, h, h, 0, 0)
        _check_cuda(c.gvxb_harris(device.h, ctypes.byref(a)))
        out = np.empty((h, w), np.uint8)
        device.download(out, dst, pitch)
        if not response:
            return out
        r = np.empty((h, w), np.float32)
        device.download(r, rsp, 4 * pitch)
        return out, r
    finally:
        device.sync()
        device.free(src), device.free(dst)
        if rsp:
            device.free(rsp)


def stencil_point(device: "Device", img: np.ndarray, mask, div: int, mode: int) -> np.ndarray:
    """Host wrapper over gvxb_stencil_point (KxK U8 stencil, mode 0 plain,
    mode 1 unsharp chain) on one U8 frame; returns the U8 result."""
    c, _ = _load()
    c.gvxb_stencil_point.argtypes = [ctypes.c_void_p, ctypes.POINTER(GvxbStencilArgs)]
    h, w = img.shape
    pitch = (w + 127) // 128 * 128
    src, dst = device.alloc(pitch * h), device.alloc(pitch * h)
    try:
        device.upload(src, pitch, np.ascontiguousarray(img, np.uint8))
        a = GvxbStencilArgs()
        a.src = GvxbImage(src, pitch, w, h, 0, 1, 0)
        a.dst = GvxbImage(dst, pitch, w, h, 0, 1, 0)
        a.ksize = int(np.asarray(mask).shape[0])
        a.mask = _mask49(mask)
        a.div_num, a.div_den, a.mode = 1, int(div), int(mode)
        a.band = GvxbBand(0, h, h, 0, 0)
        _check_cuda(c.gvxb_stencil_point(device.h, ctypes.byref(a)))
        out = np.empty((h, w), np.uint8)
        device.download(out, dst, pitch)
        device.sync()
        return out
    finally:
        device.sync()
        device.free(src), device.free(dst)


def conv_stats(device: "Device", img: np.ndarray, mask, scale: int, conv_format: int = 2, shift: int = 0,
               wrap: bool = False, bins: int = 256, offset: int = 0, rng: int = 256, one_launch: bool = False,
               repeat: int = 1):
    """Host wrapper over gvxb_conv_stats on one U8 frame: returns
    (converted U8 image, histogram int64[bins], mean, stddev).  one_launch:
    pass zeroed `work` scratch (the single-kernel form); repeat: execute
    that many times (the scratch must come back zero each time)."""
    c, _ = _load()
    c.gvxb_conv_stats.argtypes = [ctypes.c_void_p, ctypes.POINTER(GvxbConvStatsArgs)]
    h, w = img.shape
    pitch = (w + 127) // 128 * 128
    src, conv = device.alloc(pitch * h), device.alloc(pitch * h)
    aux = device.alloc(16 * bins + 64 + 32)
    work = device.alloc(8 * (bins + 1)) if one_launch else 0
    try:
        if one_launch:  # zero scratch: the sums and the accumulators
            device.upload(aux, 16 * bins + 96, np.zeros((1, 16 * bins + 96), np.uint8))
            device.upload(work, 8 * (bins + 1), np.zeros((1, 8 * (bins + 1)), np.uint8))
        device.upload(src, pitch, np.ascontiguousarray(img, np.uint8))
        a = GvxbConvStatsArgs()
        a.src = GvxbImage(src, pitch, w, h, 0, 1, 0)
        a.converted = GvxbImage(conv, pitch, w, h, 0, 1, 0)
        a.ksize = int(np.asarray(mask).shape[0])
        a.mask = _mask49(mask)
        a.scale, a.conv_format, a.shift, a.wrap = int(scale), int(conv_format), int(shift), int(wrap)
        a.bins, a.offset, a.range = int(bins), int(offset), int(rng)
        a.hist, a.sum, a.sumsq = aux, aux + 16 * bins, aux + 16 * bins + 8
        a.mean, a.stddev = aux + 16 * bins + 16, aux + 16 * bins + 32
        a.work = work or None
        for _ in range(repeat):
            _check_cuda(c.gvxb_conv_stats(device.h, ctypes.byref(a)))
        out = np.empty((h, w), np.uint8)
        device.download(out, conv, pitch)
        raw = np.empty(2 * bins + 6, np.int64)
        device.download(raw.reshape(1, -1).view(np.uint8), aux, raw.nbytes)
        device.sync()
        hist = raw[1:2 * bins:2].copy()
        mean = float(raw[2 * bins + 3:2 * bins + 4].view(np.float64)[0])
        sd = float(raw[2 * bins + 5:2 * bins + 6].view(np.float64)[0])
        return out, hist, mean, sd
    finally:
        device.sync()
        device.free(src), device.free(conv), device.free(aux)
        if work:
            device.free(work)


def band_rows(height: int, world: int, rank: int):
    c, _ = _load()
    r0, r1 = ctypes.c_int32(), ctypes.c_int32()
    _check_cuda(c.gvxb_band_rows(height, world, rank, ctypes.byref(r0), ctypes.byref(r1)))
    return r0.value, r1.value


class GvxbBandPlan(ctypes.Structure):
    """include/gvxb.h gvxb_band_plan."""
    _fields_ = [(n, ctypes.c_int32) for n in ("height", "world", "rank", "halo", "row0", "row1", "src_row0",
                                              "src_row1", "interior_row0", "interior_row1", "n_edges")] + [
        ("edge_row0", ctypes.c_int32 * 2), ("edge_row1", ctypes.c_int32 * 2), ("peer", ctypes.c_int32 * 2),
        ("send_row0", ctypes.c_int32 * 2), ("send_rows", ctypes.c_int32 * 2), ("recv_row0", ctypes.c_int32 * 2),
        ("recv_rows", ctypes.c_int32 * 2)]


def band_plan(height: int, world: int, rank: int, halo: int) -> dict:
    """gvxb_band_plan_make: rows, overlap split and exchange schedule of one band."""
    c, _ = _load()
    p = GvxbBandPlan()
    _check_cuda(c.gvxb_band_plan_make(height, world, rank, halo, ctypes.byref(p)))
    d = {n: getattr(p, n) for n, _ in GvxbBandPlan._fields_[:11]}
    d["edges"] = [(p.edge_row0[i], p.edge_row1[i]) for i in range(p.n_edges)]
    d["peers"] = [None if p.peer[s] < 0 else {"peer": p.peer[s], "send": (p.send_row0[s], p.send_row0[s] + p.send_rows[s]),
                                               "recv": (p.recv_row0[s], p.recv_row0[s] + p.recv_rows[s])}
                  for s in range(2)]
    return d


class Comm:
    """NCCL communicator of the C-ABI (gvxb_comm_*): the halo exchange and
    the max-over-ranks timing of row bands, one process per GPU.  The
    128-byte unique id travels from rank 0 through a file named after the
    launcher (torchrun agent pid + MASTER_PORT) so no Python collective
    library is needed."""

    def __init__(self, rank: int, world: int, device: int, uid: bytes | None = None, timeout: float = 120.0):
        c, _ = _load()
        self.c, self.rank, self.world = c, rank, world
        if uid is None:
            uid = self._exchange_id(rank, timeout)
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        h = ctypes.c_void_p()
        _check_cuda(c.gvxb_comm_create(device, rank, world, buf, ctypes.byref(h)))
        self.h = h

    @staticmethod
    def unique_id() -> bytes:
        c, _ = _load()
        buf = (ctypes.c_uint8 * 128)()
        _check_cuda(c.gvxb_comm_unique_id(buf))
        return bytes(buf)

    def _exchange_id(self, rank: int, timeout: float) -> bytes:
        import tempfile
        import time
        key = f"{os.getppid()}_{os.environ.get('MASTER_PORT', '0')}_{os.environ.get('TORCHELASTIC_RUN_ID', '')}"
        path = pathlib.Path(tempfile.gettempdir()) / f"gvx_nccl_id_{key}"
        if rank == 0:
            uid = self.unique_id()
            tmp = path.with_suffix(".tmp")
            tmp.write_bytes(uid)
            os.replace(tmp, path)
            self._id_path = path
            return uid
        t_end = time.time() + timeout
        while time.time() < t_end:
            if path.exists():
                data = path.read_bytes()
                if len(data) == 128:
                    return data
            time.sleep(0.01)
        raise TimeoutError(f"NCCL unique id not published at {path}")

    def allreduce_max(self, x: float) -> float:
        v = ctypes.c_double(x)
        _check_cuda(self.c.gvxb_comm_allreduce_max(self.h, ctypes.byref(v)))
        return v.value

    def barrier(self):
        _check_cuda(self.c.gvxb_comm_barrier(self.h))

    def close(self):
        if getattr(self, "_id_path", None) is not None:
            try:
                self._id_path.unlink()
            except OSError:
                pass
            self._id_path = None
        if getattr(self, "h", None):
            self.c.gvxb_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Band:
    """One row band of a ConfigGraph's plan (gvx::BandedSession through
    gvx_c.h).  Slots: 0 = input image, k >= 1 = config output k - 1."""

    def __init__(self, graph: "ConfigGraph", rank: int = 0, world: int = 1, comm: Comm | None = None,
                 device: int = -1, frames: int = 1, _handle=None):
        self.graph = graph
        if _handle is not None:
            self._h, self._own = _handle, False
        else:
            h = ctypes.c_void_p()
            _check_graph(_graph.gvxc_band_create(graph.handle, rank, world, comm.h if comm else None, device, frames,
                                                 ctypes.byref(h)))
            self._h, self._own = h, True
        v = (ctypes.c_int32 * 9)()
        _check_graph(_graph.gvxc_band_layout(self._h, v))
        self.layout = dict(zip(["rank", "world", "width", "height", "row0", "row1", "src_row0", "src_row1", "halo"],
                               list(v)))

    def close(self):
        if getattr(self, "_own", False) and getattr(self, "_h", None):
            _graph.gvxc_band_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def tensor(self, slot: int):
        """(device pointer, pitch, frame stride, first global row, rows)."""
        p, pitch, fs = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_int64()
        r0, n = ctypes.c_int32(), ctypes.c_int32()
        _check_graph(_graph.gvxc_band_tensor(self._h, slot, ctypes.byref(p), ctypes.byref(pitch), ctypes.byref(fs),
                                             ctypes.byref(r0), ctypes.byref(n)))
        return p.value, pitch.value, fs.value, r0.value, n.value

    def upload(self, slot: int, rows: np.ndarray, first_row: int, frame: int = 0):
        a = np.ascontiguousarray(rows)
        _check_graph(_graph.gvxc_band_upload(self._h, slot, a.ctypes.data, a.strides[0], first_row, a.shape[0], frame))

    def download(self, slot: int, first_row: int, rows: int, dtype, frame: int = 0) -> np.ndarray:
        out = np.empty((rows, self.layout["width"]), dtype)
        _check_graph(_graph.gvxc_band_download(self._h, slot, out.ctypes.data, out.strides[0], first_row, rows, frame))
        return out

    def set_stream(self, stream: int | None):
        _check_graph(_graph.gvxc_band_set_stream(self._h, ctypes.c_void_p(stream or 0)))

    def set_overlap(self, mode: int):
        _check_graph(_graph.gvxc_band_set_overlap(self._h, mode))

    def bind(self, slot: int, dptr: int, pitch: int, frame_stride: int = 0):
        _check_graph(_graph.gvxc_band_bind(self._h, slot, ctypes.c_void_p(dptr), pitch, frame_stride))

    def launch(self):
        _check_graph(_graph.gvxc_band_launch(self._h))

    def sync(self):
        _check_graph(_graph.gvxc_band_sync(self._h))

    def launches(self) -> int:
        return _graph.gvxc_band_launches(self._h)

    def run_host(self, src: int, src_pitch: int, slot: int, dst: int, dst_pitch: int, piece_rows: int = 1024):
        """Host pointers (ints): src = input slab rows, dst = output rows of the band."""
        _check_graph(_graph.gvxc_band_run_host(self._h, ctypes.c_void_p(src), src_pitch, slot, ctypes.c_void_p(dst),
                                               dst_pitch, piece_rows))

    def describe(self) -> str:
        buf = ctypes.create_string_buffer(8192)
        _check_graph(_graph.gvxc_band_describe(self._h, buf, len(buf)))
        return buf.value.decode()


class BandGroup:
    """n row bands of one image in this process (gvx::BandGroup): band i on
    devices[i]; halo rows by strided peer copies."""

    def __init__(self, graph: "ConfigGraph", devices, frames: int = 1):
        self.graph = graph
        devs = (ctypes.c_int * len(devices))(*devices)
        h = ctypes.c_void_p()
        _check_graph(_graph.gvxc_group_create(graph.handle, len(devices), devs, frames, ctypes.byref(h)))
        self._h = h
        self.bands = []
        for i in range(len(devices)):
            bh = ctypes.c_void_p()
            _check_graph(_graph.gvxc_group_band(h, i, ctypes.byref(bh)))
            self.bands.append(Band(graph, _handle=bh))

    def launch(self):
        _check_graph(_graph.gvxc_group_launch(self._h))

    def sync(self):
        _check_graph(_graph.gvxc_group_sync(self._h))

    def close(self):
        if getattr(self, "_h", None):
            for b in self.bands:
                b._h = None
            _graph.gvxc_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class HostBuffer:
    """Page-locked host memory (gvxb_host_alloc) viewed as a numpy array."""

    def __init__(self, shape, dtype):
        c, _ = _load()
        self.c = c
        n = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = ctypes.c_void_p()
        _check_cuda(c.gvxb_host_alloc(max(n, 1), ctypes.byref(p)))
        self.ptr = p.value
        buf = (ctypes.c_uint8 * n).from_address(self.ptr)
        self.array = np.frombuffer(buf, dtype=dtype).reshape(shape)

    def close(self):
        if getattr(self, "ptr", None):
            self.array = None
            self.c.gvxb_host_free(ctypes.c_void_p(self.ptr))
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


__all__ = ["GraphvxError", "ConfigGraph", "Session", "Device", "build", "device_count", "random_u8",
           "stencil_point", "conv_stats", "harris", "GraphFile", "json_roundtrip", "parse_outputs", "Pipeline",
           "band_rows", "band_plan", "Band", "BandGroup", "Comm", "HostBuffer", "libraries", "CONFIG_SIZE", "CONFIG_SEED", "CONFIG_FRAMES"]
