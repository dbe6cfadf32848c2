"""B200-native Sliding Window Recurrence (Block Two-Pass) and Phalanx mixer.

Hot path of arXiv 2512.13921 as a C-ABI library (``libswr.so``, include/swr.h)
of hand-written sm_100a CUDA kernels, with a thin Python binding.

    from paper_2512_13921_b200 import swr, mix, swr_fwd, swr_bwd, phalanx_mix, phalanx_mix_bwd
"""
from . import _lib  # noqa: F401  (fails loudly if libswr.so is missing)
from ._lib import SWR_PATH_AUTO, SWR_PATH_FFMA, SWR_PATH_TC, SwrError, launch_count, last_path, set_path  # noqa: F401
from .ops import (DecodeState, layout_copies, layer_mix, phalanx_layer_mix, phalanx_layer_mix_bwd, mix, phalanx_mix, phalanx_mix_bwd, phalanx_mix_decode_step, swr,  # noqa: F401
                  swr_bwd, swr_decode_step, swr_exact, swr_exact_bwd, swr_exact_fwd, swr_fwd, swr_uniform_fwd)

ELL = 16  # block length
