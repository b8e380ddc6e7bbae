"""B200-native TFLA (Tiled Flash Linear Attention) for mLSTMexp / mLSTMsig."""
from . import _ffi  # noqa: F401
