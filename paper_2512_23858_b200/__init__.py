"""B200-native Yggdrasil speculative-decoding step (reference: arxiv 2512.23858 ``specsim``).

Host side in Python/PyTorch; every hot op runs in hand-written sm_100a CUDA (libygg.so,
C ABI in include/ygg.h).  There is no CPU fallback: importing works anywhere, but any call
that reaches the device path raises unless a B200 and the built library are present.
"""

__version__ = "0.1.0"
