"""ctypes binding of the sdb200 C-ABI (include/sdb200.h) in `_sdb200.so`.

There is no fallback: if the library is missing, or no CUDA device is
present, calls raise `NativeUnavailable` -- the product path never computes on
the CPU.  PyTorch is used only for device memory and streams; every call
passes raw device pointers and the current CUDA stream.
"""

from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "_sdb200.so")

_c_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_sz = ctypes.c_size_t

# name -> (restype, argtypes); must mirror include/sdb200.h exactly.
SIGNATURES = {
    "sdb_version": (ctypes.c_int, []),
    "sdb_chain_fb_f64_workspace": (_sz, [_i64, _i32, _i32]),
    "sdb_chain_fb_f64": (ctypes.c_int, [_c_p, _c_p, _i64, _i32, _i32, _c_p, _c_p, _c_p, _c_p, _c_p, _sz, _c_p]),
    "sdb_semimarkov_fb_f64_workspace": (_sz, [_i64, _i32, _i32, _i32]),
    "sdb_semimarkov_fb_f64": (ctypes.c_int, [_c_p, _i64, _i32, _i32, _i32, _c_p, _c_p, _c_p, _c_p, _sz, _c_p]),
    "sdb_nw_fb_f64_workspace": (_sz, [_i64, _i32, _i32]),
    "sdb_nw_fb_f64": (ctypes.c_int, [_c_p, _i64, _i32, _i32, _c_p, _c_p, _c_p, _c_p, _sz, _c_p]),
    "sdb_ctc_fb_f64_workspace": (_sz, [_i64, _i32, _i32, _i32]),
    "sdb_ctc_fb_f64": (ctypes.c_int, [_c_p, _c_p, _i64, _i32, _i32, _i32, _c_p, _c_p, _c_p, _c_p, _sz, _c_p]),
    "sdb_tree_fb_f64_workspace": (_sz, [_i64, _i32, _i32]),
    "sdb_tree_fb_f64": (ctypes.c_int, [_c_p, _i64, _i32, _i32, _c_p, _c_p, _c_p, _c_p, _sz, _c_p]),
    "sdb_pcfg_f64_workspace": (_sz, [_i64, _i32, _i32, _i32, _i32]),
    "sdb_pcfg_f64": (ctypes.c_int, [_c_p, _c_p, _c_p, _c_p, _i64, _i32, _i32, _i32, _c_p, _c_p, _c_p, _c_p, _c_p,
                                    _c_p, _c_p, _sz, _c_p]),
    "sdb_pcfg_viterbi_f64": (ctypes.c_int, [_c_p, _c_p, _c_p, _c_p, _i64, _i32, _i32, _i32, _c_p, _c_p, _c_p, _c_p,
                                            _sz, _c_p]),
    "sdb_mtt_f64_workspace": (_sz, [_i64, _i32]),
    "sdb_mtt_f64": (ctypes.c_int, [_c_p, _i64, _i32, _i32, _c_p, _c_p, _c_p, _c_p, _sz, _c_p]),
    "sdb_eisner_f64": (ctypes.c_int, [_c_p, _i64, _i32, _i32, _c_p, _c_p, _c_p, _c_p]),
    "sdb_masked_dot_f64": (ctypes.c_int, [_c_p, _c_p, _i64, _i64, _c_p, _c_p, _c_p]),
    "sdb_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "sdb_last_cuda_error": (ctypes.c_char_p, []),
    "sdb_chain_fb_workspace": (_sz, [_i64, _i32, _i32]),
    "sdb_chain_fb": (ctypes.c_int, [_c_p, _c_p, _i64, _i32, _i32, _c_p, _c_p, _c_p, _c_p, _c_p, _sz, _c_p]),
    "sdb_chain_viterbi_workspace": (_sz, [_i64, _i32, _i32]),
    "sdb_chain_viterbi": (ctypes.c_int, [_c_p, _c_p, _i64, _i32, _i32, _c_p, _c_p, _c_p, _c_p, _sz, _c_p]),
    "sdb_nw_fb_workspace": (_sz, [_i64, _i32, _i32]),
    "sdb_nw_fb": (ctypes.c_int, [_c_p, _i64, _i32, _i32, _c_p, _c_p, _c_p, _c_p, _sz, _c_p]),
    "sdb_nw_viterbi_workspace": (_sz, [_i64, _i32, _i32]),
    "sdb_nw_viterbi": (ctypes.c_int, [_c_p, _i64, _i32, _i32, _c_p, _c_p, _c_p, _c_p, _sz, _c_p]),
    "sdb_ctc_fb_workspace": (_sz, [_i64, _i32, _i32, _i32]),
    "sdb_ctc_fb": (ctypes.c_int, [_c_p, _c_p, _i64, _i32, _i32, _i32, _c_p, _c_p, _c_p, _c_p, _sz, _c_p]),
    "sdb_ctc_viterbi_workspace": (_sz, [_i64, _i32, _i32, _i32]),
    "sdb_ctc_viterbi": (ctypes.c_int, [_c_p, _c_p, _i64, _i32, _i32, _i32, _c_p, _c_p, _c_p, _c_p, _sz, _c_p]),
    "sdb_tree_fb_workspace": (_sz, [_i64, _i32, _i32]),
    "sdb_tree_fb": (ctypes.c_int, [_c_p, _i64, _i32, _i32, _c_p, _c_p, _c_p, _c_p, _sz, _c_p]),
    "sdb_tree_viterbi": (ctypes.c_int, [_c_p, _i64, _i32, _i32, _c_p, _c_p, _c_p, _c_p]),
    "sdb_mtt": (ctypes.c_int, [_c_p, _i64, _i32, _i32, _c_p, _c_p, _c_p, _c_p]),
    "sdb_eisner": (ctypes.c_int, [_c_p, _i64, _i32, _i32, _c_p, _c_p, _c_p, _c_p]),
    "sdb_kuhlmann": (ctypes.c_int, [_c_p, _i64, _i32, _i32, _c_p, _c_p, _c_p, _c_p]),
    "sdb_pcfg_fb_workspace": (_sz, [_i64, _i32, _i32, _i32]),
    "sdb_pcfg_fb": (ctypes.c_int, [_c_p, _c_p, _c_p, _c_p, _i64, _i32, _i32, _i32, _c_p, _c_p, _c_p, _c_p, _sz,
                                   _c_p]),
    "sdb_pcfg_grad_workspace": (_sz, [_i64, _i32, _i32, _i32]),
    "sdb_pcfg_grad": (ctypes.c_int, [_c_p, _c_p, _c_p, _c_p, _i64, _i32, _i32, _i32, _c_p, _c_p, _c_p, _c_p, _c_p,
                                     _c_p, _c_p, _sz, _c_p]),
    "sdb_pcfg_viterbi_workspace": (_sz, [_i64, _i32, _i32, _i32]),
    "sdb_pcfg_viterbi": (ctypes.c_int, [_c_p, _c_p, _c_p, _c_p, _i64, _i32, _i32, _i32, _c_p, _c_p, _c_p, _c_p,
                                        _sz, _c_p]),
    "sdb_chain_sample_workspace": (_sz, [_i64, _i32, _i32]),
    "sdb_chain_sample": (ctypes.c_int, [_c_p, _c_p, _i64, _i32, _i32, _c_p, _i64, _i32, _c_p, _c_p, _c_p, _c_p, _sz,
                                        _c_p]),
    "sdb_nw_sample_workspace": (_sz, [_i64, _i32, _i32]),
    "sdb_nw_sample": (ctypes.c_int, [_c_p, _i64, _i32, _i32, _c_p, _i64, _i32, _c_p, _c_p, _c_p, _c_p, _sz, _c_p]),
    "sdb_ctc_sample_workspace": (_sz, [_i64, _i32, _i32, _i32]),
    "sdb_ctc_sample": (ctypes.c_int, [_c_p, _c_p, _i64, _i32, _i32, _i32, _c_p, _i64, _i32, _c_p, _c_p, _c_p, _c_p,
                                      _sz, _c_p]),
    "sdb_tree_sample_workspace": (_sz, [_i64, _i32, _i32]),
    "sdb_tree_sample": (ctypes.c_int, [_c_p, _i64, _i32, _i32, _c_p, _i64, _i32, _c_p, _c_p, _c_p, _c_p, _sz, _c_p]),
    "sdb_eisner_decode_workspace": (_sz, [_i64, _i32]),
    "sdb_eisner_decode": (ctypes.c_int, [_c_p, _i64, _i32, _i32, _c_p, _i64, _i32, _c_p, _c_p, _c_p, _c_p, _sz,
                                         _c_p]),
    "sdb_cle_workspace": (_sz, [_i64, _i32]),
    "sdb_cle": (ctypes.c_int, [_c_p, _i64, _i32, _i32, _c_p, _c_p, _c_p, _sz, _c_p]),
    "sdb_wilson_workspace": (_sz, [_i64, _i32]),
    "sdb_wilson_begin": (ctypes.c_int, [_i64, _i32, _c_p, _c_p, _c_p, _c_p, _sz, _c_p]),
    "sdb_wilson_step": (ctypes.c_int, [_c_p, _i64, _i32, _c_p, _i64, _i64, _c_p, _c_p, _c_p, _c_p, _sz, _c_p]),
    "sdb_semimarkov_sample_workspace": (_sz, [_i64, _i32, _i32, _i32]),
    "sdb_semimarkov_sample": (ctypes.c_int, [_c_p, _i64, _i32, _i32, _i32, _c_p, _i64, _i32, _c_p, _c_p, _c_p, _c_p,
                                             _c_p, _sz, _c_p]),
    "sdb_pcfg_sample": (ctypes.c_int, [_c_p, _c_p, _c_p, _c_p, _i64, _i32, _i32, _i32, _c_p, _i64, _i32, _c_p, _c_p,
                                       _c_p, _c_p, _sz, _c_p]),
    "sdb_mtt_ex_workspace": (_sz, [_i64, _i32]),
    "sdb_mtt_ex": (ctypes.c_int, [_c_p, _i64, _i32, _i32, _c_p, _c_p, _c_p, _c_p, _sz, _c_p]),
    "sdb_chain_fb_lengths": (ctypes.c_int, [_c_p, _c_p, _c_p, _i64, _i32, _i32, _c_p, _c_p, _c_p, _c_p, _c_p, _sz,
                                            _c_p]),
    "sdb_chain_viterbi_lengths": (ctypes.c_int, [_c_p, _c_p, _c_p, _i64, _i32, _i32, _c_p, _c_p, _c_p, _c_p]),
    "sdb_masked_dot": (ctypes.c_int, [_c_p, _c_p, _i64, _i64, _c_p, _c_p, _c_p]),
    "sdb_semimarkov_fb": (ctypes.c_int, [_c_p, _i64, _i32, _i32, _i32, _c_p, _c_p, _c_p, _c_p]),
    "sdb_semimarkov_viterbi_workspace": (_sz, [_i64, _i32, _i32, _i32]),
    "sdb_semimarkov_viterbi": (ctypes.c_int, [_c_p, _i64, _i32, _i32, _i32, _c_p, _c_p, _c_p, _c_p, _c_p, _sz,
                                              _c_p]),
}


class NativeUnavailable(RuntimeError):
    """The sm_100a library or the CUDA device is missing (no CPU fallback)."""


class NativeError(RuntimeError):
    """A C-ABI call returned a negative SDB_ERR_* code."""


_lib = None


def load():
    """Load `_sdb200.so` (no device needed; used by the symbol tests)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailable(
            f"{LIB_PATH} not built; run `python -m paper_2308_03291_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str):
    if rc != 0:
        lib = load()
        msg = lib.sdb_status_string(rc).decode()
        if rc == -3:  # SDB_ERR_CUDA: add the runtime's own message
            msg += ": " + lib.sdb_last_cuda_error().decode()
        raise NativeError(f"{what}: {msg} (code {rc})")
