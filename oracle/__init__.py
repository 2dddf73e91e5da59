"""ORACLE — test infrastructure only.

Python access to the CPU checkers:
  * ``ref``  : the unmodified reference engine (oracle/_ref/liboracle_ref.so,
               built from /root/reference by oracle/Makefile with
               -Dgvx=gvxref) — run_naive on the five configurations;
  * ``port`` : the plain-C restatement oracle/gvx_oracle.c
               (oracle/build/libgvx_oracle.so).
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline /
--impl reference legs may import this package; the product never does.
"""
from __future__ import annotations

import ctypes
import pathlib
import subprocess

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
REF_LIB = HERE / "_ref" / "liboracle_ref.so"
PORT_LIB = HERE / "build" / "libgvx_oracle.so"
REFERENCE_SRC = pathlib.Path("/root/reference/proj")

_ref = None
_port = None


def build() -> None:
    """Build the port always; the reference oracle only where /root/reference exists."""
    subprocess.run(["make", "-C", str(HERE), "oracle"], check=True, capture_output=True)
    if REFERENCE_SRC.exists():
        subprocess.run(["make", "-j8", "-C", str(HERE), "ref"], check=True, capture_output=True)


def have_ref() -> bool:
    return REF_LIB.exists()


def ref():
    global _ref
    if _ref is None:
        if not REF_LIB.exists():
            raise FileNotFoundError(f"{REF_LIB} not built (needs /root/reference; see oracle/Makefile)")
        lib = ctypes.CDLL(str(REF_LIB))
        lib.oref_last_error.restype = ctypes.c_char_p
        lib.oref_random_image.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_ulonglong, ctypes.c_void_p]
        lib.oref_run_config.argtypes = [ctypes.c_int] * 3 + [ctypes.c_void_p] * 2 + [
            ctypes.POINTER(ctypes.c_longlong), ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
        lib.oref_config_counters.argtypes = [ctypes.c_int] * 3 + [ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong)]
        lib.oref_have_graph_io.restype = ctypes.c_int
        if lib.oref_have_graph_io():
            SZ = ctypes.c_size_t
            lib.oref_json_roundtrip.argtypes = [ctypes.c_char_p, ctypes.c_char_p, SZ, ctypes.POINTER(SZ)]
            lib.oref_json_run.argtypes = [ctypes.c_char_p, ctypes.c_ulonglong, ctypes.c_void_p, SZ,
                                          ctypes.POINTER(SZ), ctypes.POINTER(ctypes.c_longlong)]
        _ref = lib
    return _ref


def have_ref_graph_io() -> bool:
    return have_ref() and bool(ref().oref_have_graph_io())


def ref_json_roundtrip(text: str) -> str:
    """The reference's save_graph_json(load_graph_json(text))."""
    lib = ref()
    need = ctypes.c_size_t()
    if lib.oref_json_roundtrip(text.encode(), None, 0, ctypes.byref(need)):
        raise RuntimeError(lib.oref_last_error().decode())
    buf = ctypes.create_string_buffer(need.value)
    lib.oref_json_roundtrip(text.encode(), buf, need.value, ctypes.byref(need))
    return buf.value.decode()


def ref_json_run(text: str, seed: int):
    """The reference pipeline over a graph file (run_naive); returns the raw
    serialised outputs and the event counters."""
    lib = ref()
    need = ctypes.c_size_t()
    counters = (ctypes.c_longlong * 4)()
    if lib.oref_json_run(text.encode(), seed, None, 0, ctypes.byref(need), counters):
        raise RuntimeError(lib.oref_last_error().decode())
    buf = (ctypes.c_uint8 * max(1, need.value))()
    lib.oref_json_run(text.encode(), seed, buf, need.value, ctypes.byref(need), counters)
    return bytes(buf)[:need.value], list(counters)


def port():
    global _port
    if _port is None:
        if not PORT_LIB.exists():
            build()
        lib = ctypes.CDLL(str(PORT_LIB))
        V = ctypes.c_void_p
        lib.gvxo_edge.argtypes = [V, ctypes.c_int, ctypes.c_int, V]
        lib.gvxo_harris.argtypes = [V, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double, V, V]
        lib.gvxo_unsharp.argtypes = [V, ctypes.c_int, ctypes.c_int, V]
        lib.gvxo_conv_stats.argtypes = [V, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_longlong),
                                        ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
        I = ctypes.c_int
        lib.gvxo_stencil_u8.argtypes = [V, I, I, I, V, ctypes.c_longlong, I, V]
        lib.gvxo_conv_stats_ex.argtypes = [V, I, I, I, V, ctypes.c_longlong, I, I, I, I, I, ctypes.c_longlong,
                                           ctypes.c_longlong, V, ctypes.POINTER(ctypes.c_double),
                                           ctypes.POINTER(ctypes.c_double), V]
        _port = lib
    return _port


def port_harris(img: np.ndarray, k: float, threshold: float):
    """gvxo_harris with explicit k / T: (U8 mask, F32 response)."""
    img = np.ascontiguousarray(img, np.uint8)
    mask = np.empty_like(img)
    resp = np.empty(img.shape, np.float32)
    port().gvxo_harris(img.ctypes.data, img.shape[1], img.shape[0], k, threshold, mask.ctypes.data,
                       resp.ctypes.data)
    return mask, resp


def port_stencil(img: np.ndarray, mask, div: int, mode: int) -> np.ndarray:
    """gvxo_stencil_u8: KxK local node sat_U8(s * (1/div)) [-> unsharp chain]."""
    img = np.ascontiguousarray(img, np.uint8)
    m = np.ascontiguousarray(mask, np.int32)
    out = np.empty_like(img)
    port().gvxo_stencil_u8(img.ctypes.data, img.shape[1], img.shape[0], m.shape[0], m.ctypes.data, div, mode,
                           out.ctypes.data)
    return out


def port_conv_stats(img: np.ndarray, mask, scale: int, conv_lo: int = -32768, conv_hi: int = 32767,
                    shift: int = 0, wrap: bool = False, bins: int = 256, offset: int = 0, rng: int = 256):
    """gvxo_conv_stats_ex: (converted U8, hist, mean, stddev)."""
    img = np.ascontiguousarray(img, np.uint8)
    m = np.ascontiguousarray(mask, np.int32)
    conv = np.empty_like(img)
    hist = np.zeros(bins, np.int64)
    mean, sd = ctypes.c_double(), ctypes.c_double()
    port().gvxo_conv_stats_ex(img.ctypes.data, img.shape[1], img.shape[0], m.shape[0], m.ctypes.data, scale,
                              conv_lo, conv_hi, shift, int(wrap), bins, offset, rng, hist.ctypes.data,
                              ctypes.byref(mean), ctypes.byref(sd), conv.ctypes.data)
    return conv, hist, mean.value, sd.value


HARRIS_K = 0.04
HARRIS_T = 1.0e9


def ref_random_u8(w: int, h: int, seed: int) -> np.ndarray:
    out = np.empty((h, w), np.uint8)
    if ref().oref_random_image(w, h, 0, seed, out.ctypes.data) != 0:
        raise RuntimeError(ref().oref_last_error().decode())
    return out


def ref_run(cfg: int, img: np.ndarray):
    """Reference run_naive on config `cfg`; returns (result, seconds)."""
    h, w = img.shape
    img = np.ascontiguousarray(img, np.uint8)
    hist = (ctypes.c_longlong * 256)()
    stats = (ctypes.c_double * 2)()
    secs = ctypes.c_double()
    out = None
    if cfg in (1, 5):
        out = np.empty((h, w), np.int16)
    elif cfg in (2, 3):
        out = np.empty((h, w), np.uint8)
    rc = ref().oref_run_config(cfg, w, h, img.ctypes.data, None if out is None else out.ctypes.data, hist, stats,
                               ctypes.byref(secs))
    if rc != 0:
        raise RuntimeError(ref().oref_last_error().decode())
    if cfg == 4:
        return (np.array(list(hist), np.int64), stats[0], stats[1]), secs.value
    return out, secs.value


def ref_counters(cfg: int, img: np.ndarray) -> dict:
    h, w = img.shape
    c = (ctypes.c_longlong * 4)()
    if ref().oref_config_counters(cfg, w, h, np.ascontiguousarray(img, np.uint8).ctypes.data, c) != 0:
        raise RuntimeError(ref().oref_last_error().decode())
    return dict(zip(["kernel_launches", "pixels_read", "pixels_written", "transfers_executed"], list(c)))


def port_run(cfg: int, img: np.ndarray):
    """The C restatement on config `cfg`."""
    lib = port()
    h, w = img.shape
    img = np.ascontiguousarray(img, np.uint8)
    if cfg in (1, 5):
        out = np.empty((h, w), np.int16)
        lib.gvxo_edge(img.ctypes.data, w, h, out.ctypes.data)
        return out
    if cfg == 2:
        out = np.empty((h, w), np.uint8)
        lib.gvxo_harris(img.ctypes.data, w, h, HARRIS_K, HARRIS_T, out.ctypes.data, None)
        return out
    if cfg == 3:
        out = np.empty((h, w), np.uint8)
        lib.gvxo_unsharp(img.ctypes.data, w, h, out.ctypes.data)
        return out
    hist = (ctypes.c_longlong * 256)()
    m, s = ctypes.c_double(), ctypes.c_double()
    lib.gvxo_conv_stats(img.ctypes.data, w, h, hist, ctypes.byref(m), ctypes.byref(s))
    return np.array(list(hist), np.int64), m.value, s.value
