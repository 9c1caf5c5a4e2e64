"""ctypes binding of libmvb.so (include/mvb.h).

The library is the only compute backend.  Loading fails loudly when the
shared object is missing, and every call checks that a CUDA device is
present; there is no CPU path behind any function of this package.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# MVB_LIB=checked loads the bounds-checked build (libmvb_checked.so, make
# checked): same ABI, counters read by check_violations()
LIB_PATH = os.path.join(_HERE, "libmvb_checked.so" if os.environ.get("MVB_LIB") == "checked"
                        else "libmvb.so")
LIB_PATH = os.environ.get("MVB_LIB_PATH", LIB_PATH)  # A/B of another build (diagnostics)

_lock = threading.Lock()
_lib = None

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
INT = ctypes.c_int
DBL = ctypes.c_double

# name -> argtypes (all return int status unless listed in _RESTYPE)
_SIGS = {
    "mvb_abi_version": [],
    "mvb_last_error": [],
    "mvb_device_info": [P, P, P],
    "mvb_struct_sizes": [P, P, P, P],
    "mvb_copy_batch": [P, P, P, I64, P, INT, P],
    "mvb_distance_streams": [P, P, P, P, I64, I64, P, P],
    "mvb_accumulate_images": [P, I64, P, I64, I64, P, P, I64, I64, I64, P],
    "mvb_upsample_streams": [P, I64, I64, P, I64, I64, I64, P, P],
    "mvb_branch_filter": [P, I64, P, I64, I64, P, P],
    "mvb_image_count": [INT],
    "mvb_enumerate": [P, P, I64, INT, P, P, P, P, P, P, P],
    "mvb_build_images": [P, P, P, I64, P, I64, P, I64, P, I64, P, P, I64, P, I64, P, P],
    "mvb_coarse_distances": [P, P, I64, I64, P, P, DBL, P, P, P, P],
    "mvb_track_bounds": [P, P, I64, P, P, P, P, P, P],
    "mvb_path_bbox": [P, I64, P, P, P],
    "mvb_finalize_lengths": [P, I64, P, P, P, P],
    "mvb_track_max": [P, P, I64, P, P, P, DBL, P, P, P, P, P],
    "mvb_gather_images": [P, P, I64, P, P],
    "mvb_track_coeffs": [P, P, I64, I64, P, P, P, P, P],
    "mvb_track_coeffs_windowed": [P, P, I64, I64, P, P, P, P, P],
    "mvb_sort_keys": [P, P, I64, I64, I64, I64, P, P, P, P],
    "mvb_delay_sort": [P, P, I64, I64, I64, I64, P, P, I64, P, P],
    "mvb_delay_sort_runs": [P, P, I64, I64, I64, I64, P, P, I64, I64, P, P],
    "mvb_delay_sort_keyed": [P, P, I64, I64, I64, I64, P, P, I64, I64, P, P, P],
    "mvb_branch_records_f32": [P, P, P, P, P, P, I64, I64, P, INT, INT, INT, P, P],
    "mvb_synthesize_f32": [P, P, I64, P, P, P, P, P, P, INT, INT, P],
    "mvb_synthesize_f32_ranged": [P, P, I64, P, P, I64, I64, INT, P, P, P, P, P, P, INT, INT, P],
    "mvb_synthesize_f32_tex": [P, P, I64, P, P, I64, I64, INT, P, P, P, I64, P, P, P, INT, INT, P],
    "mvb_reduce_partials_f32": [P, I64, I64, P, P, P],
    "mvb_synthesize_f64": [P, I64, I64, P, P, P, P, P, P, P],
    "mvb_synthesize_f64_ex": [P, I64, I64, P, P, P, P, P, P, I64, P],
    "mvb_energy_index": [P, I64, I64, DBL, P, P],
    "mvb_decimate_rows": [P, P, I64, I64, I64, P, P],
    "mvb_spectrum_index": [P, I64, I64, DBL, P, P, P],
    "mvb_center_paths": [P, I64, I64, P, P, P],
    "mvb_static_taps": [P, P, P, I64, P, I64, P, DBL, DBL, DBL, P, P, P, P],
    "mvb_static_gather": [P, P, P, I64, I64, P, I64, P, P],
    "mvb_block_convolve": [P, I64, I64, I64, I64, INT, P, P, I64, I64, P, I64, P],
    "mvb_splice_sum": [P, I64, I64, I64, I64, I64, P, I64, P, I64, P],
    "mvb_signal_plane_f32": [P, P, P, P, I64, I64, P, P],
    "mvb_render_tracks_and_synthesize": [P, P, I64, P, P],
    "mvb_synthesize_f32_table": [P, P, I64, P, P, P, P, P, P, P, INT, P],
    "mvb_check_violations": [P, INT],
    "mvb_fft_scratch_elems": [I64, I64],
    "mvb_fft_c2c": [P, I64, I64, INT, P, P],
    "mvb_path_spectrum_scratch": [I64, I64],
    "mvb_path_spectrum_index": [P, I64, I64, DBL, P, P, P],
    "mvb_lowpass_scratch": [I64, I64],
    "mvb_lowpass_paths": [P, I64, I64, DBL, DBL, P, P, P],
    "mvb_peak_ffma": [INT, INT, P, P],
    "mvb_peak_dfma": [INT, INT, P, P],
    "mvb_peak_l1": [INT, INT, P, P, P],
}
_RESTYPE = {"mvb_last_error": ctypes.c_char_p, "mvb_image_count": I64,
            "mvb_fft_scratch_elems": I64, "mvb_path_spectrum_scratch": I64,
            "mvb_lowpass_scratch": I64}

# kernels launched by one successful call (entry points not listed launch
# one; the query functions launch none) -- feeds launch_count()
_KERNELS = {"mvb_track_max": 2, "mvb_path_bbox": 2, "mvb_center_paths": 2,
            "mvb_spectrum_index": 2, "mvb_abi_version": 0, "mvb_last_error": 0,
            "mvb_device_info": 0, "mvb_struct_sizes": 0, "mvb_copy_batch": 0, "mvb_image_count": 0,
            "mvb_check_violations": 0, "mvb_fft_scratch_elems": 0,
            "mvb_path_spectrum_scratch": 0, "mvb_lowpass_scratch": 0}
_launches = 0

IMAGE_BYTES, JOB_BYTES, WORK_BYTES, COEF_BYTES = 96, 152, 32, 48


MAX_CLASSES = 8
DELAY_SORT_MAX = 16384  # mvb.h MVB_DELAY_SORT_MAX
EXACT_LIST_WORDS = 16386  # mvb.h MVB_EXACT_LIST_WORDS (mvb_track_max scratch)
SPEC_PARTS = 256  # mvb.h MVB_SPEC_PARTS (mvb_center_paths / mvb_spectrum_index scratch)


class ClassTable(ctypes.Structure):
    """mvb_class_table (mvb.h): image classes of one job group."""

    _fields_ = [("n", ctypes.c_int32), ("factor", ctypes.c_int32 * MAX_CLASSES),
                ("fit", ctypes.c_int32 * MAX_CLASSES), ("count", ctypes.c_int32 * MAX_CLASSES),
                ("table", ctypes.c_int64 * MAX_CLASSES), ("sel_off", ctypes.c_int64 * MAX_CLASSES)]


_P, _D, _I32, _I64 = ctypes.c_void_p, ctypes.c_double, ctypes.c_int32, ctypes.c_int64


class RenderArgs(ctypes.Structure):
    """mvb_render_args (mvb.h): one job of mvb_render_tracks_and_synthesize."""

    _fields_ = [("d_signal", _P), ("n_signal", _I64), ("d_pos", _P), ("T", _I64),
                ("d_mic", _P), ("mic_moving", _I32), ("max_order", _I32),
                ("dims", _D * 3), ("walls", _D * 6), ("n_tiers", _I32),
                ("tier_order", _I32 * MAX_CLASSES), ("tier_factor", _I32 * MAX_CLASSES),
                ("d_coarse_pos", _P * MAX_CLASSES), ("d_coarse_mic", _P * MAX_CLASSES),
                ("h_phase_table", _P * MAX_CLASSES), ("h_branches", _P),
                ("poly_order", _I32), ("branch_len", _I32), ("nominal_delay", _I32),
                ("rate", _D), ("c", _D), ("d_min", _D)]


class MvbError(RuntimeError):
    """A libmvb call returned a non-zero status."""


def lib():
    """Load libmvb.so once; raise if it is absent (no fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise MvbError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (nvcc, sm_100a). This package has no CPU implementation.")
        L = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = _RESTYPE.get(name, ctypes.c_int)
        sizes = [ctypes.c_int() for _ in range(4)]
        L.mvb_struct_sizes(*[ctypes.byref(s) for s in sizes])
        got = tuple(s.value for s in sizes)
        if got != (IMAGE_BYTES, JOB_BYTES, WORK_BYTES, COEF_BYTES):
            raise MvbError(f"libmvb struct layout mismatch: {got}")
        _lib = L
    return _lib


def call(name: str, *args) -> None:
    """Invoke a status-returning entry point; raise MvbError on failure."""
    global _launches
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        msg = lib().mvb_last_error().decode("utf-8", "replace")
        raise MvbError(f"{name} failed ({rc}): {msg}")
    _launches += _KERNELS.get(name, 1)


def check_violations():
    """Per-check violation counters of the checked build (reset on read), or
    None for the normal build."""
    buf = (ctypes.c_int64 * 16)()
    n = lib().mvb_check_violations(buf, 16)
    return None if n < 0 else [int(buf[i]) for i in range(n)]


def launch_count() -> int:
    """libmvb kernels launched by this process so far (zero-sized calls
    that return early are counted too: an upper bound by a few)."""
    return _launches


def image_count(max_order: int) -> int:
    return int(lib().mvb_image_count(int(max_order)))


def device_info():
    sm, ma, mi = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    call("mvb_device_info", ctypes.byref(sm), ctypes.byref(ma), ctypes.byref(mi))
    return sm.value, ma.value, mi.value


def loaded_path() -> str | None:
    return LIB_PATH if _lib is not None else None
