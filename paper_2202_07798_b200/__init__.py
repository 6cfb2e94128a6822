"""B200-native trainer / predictor for BB-ML's Poisson NN and BR-BPNN
(arXiv 2202.07798), a drop-in for the reference ``bbcount`` hot path.

Compute runs only in the sm_100a kernels of ``libbbml.so`` (C-ABI in
``include/bbml.h``); there is no CPU fallback.
"""

__version__ = "0.1.0"
