"""B200-native batched MAP (forward-backward) decoder for q-ary synchronization
codes over the BSID channel (arXiv 1802.08483).

The hot path lives in ``libbsidmap.so`` (hand-written CUDA for sm_100a behind
the C ABI of ``include/bsidmap.h``); this package only marshals arguments.
PyTorch supplies device memory, streams and process groups.
"""
from .decoder import Decoder, drift_limits, drift_pmf, phi, state_space  # noqa: F401
from . import _lib  # noqa: F401

MODE_AUTO = _lib.BSIDMAP_MODE_AUTO
MODE_STORED = _lib.BSIDMAP_MODE_STORED
MODE_RECOMPUTE = _lib.BSIDMAP_MODE_RECOMPUTE
MODE_GAMMASUM = _lib.BSIDMAP_MODE_GAMMASUM
FRAME_OK = _lib.BSIDMAP_FRAME_OK
FRAME_DRIFT_OUT_OF_RANGE = _lib.BSIDMAP_FRAME_DRIFT_OUT_OF_RANGE
FRAME_UNDERFLOW = _lib.BSIDMAP_FRAME_UNDERFLOW
