"""paper_2011_13695_b200 — B200-native (sm_100a) block-wise optical-receiver DSP chain of
arXiv 2011.13695 (van der Heide et al., JLT 2021) behind the C ABI of include/rx.h.

The product path is librx.so (hand-written CUDA in csrc/) plus the ctypes binding in rx.py.
There is no CPU fallback: importing works without a GPU, but every call needs librx.so and
a CUDA device.
"""
from .rx import (  # noqa: F401
    FLAGS,
    KCLASSES,
    PROBES,
    RX_IN_F32,
    RX_IN_U12_PACKED,
    RX_IN_U12_IN_U16,
    RX_PAM,
    RX_QAM_KK,
    Receiver,
    RxConfig,
    RxError,
    RxStats,
    Transmitter,
    TxConfig,
    default_config,
    load,
)
