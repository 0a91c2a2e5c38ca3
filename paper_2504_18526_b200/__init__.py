"""B200-native SI-MLSDC / DG-SEM sweep path (arXiv 2504.18526 hot path).

Drop-in GPU replacement for the reference package's problem / operator /
sweeper / level API (``sisdc.dgsem``, ``sisdc.sdc``, ``sisdc.mlsdc``,
``sisdc.transfer``, ``sisdc.collocation``).  All arithmetic on the path runs
in hand-written sm_100a CUDA kernels in ``libsisdc_b200.so`` (``csrc/``),
reached through the C ABI in ``include/sisdc_b200.h``.
"""
__version__ = "0.1.0"
