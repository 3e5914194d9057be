"""B200-native decentralized Wiener-filter precoding (arXiv 1804.10987).

The hot path (PD-WF and FD-WF per subcarrier and cluster: Gram, cross-cluster
sum, regularised Cholesky solve, Lemma-1 beta, precode x_c = H_c^H z) runs in
hand-written sm_100a CUDA kernels behind the C-ABI of libdp.so
(include/dp.h).  `Precoder` is the torch-facing wrapper; `_lib` is the
same-name ctypes binding.  Importing this package does not load libdp.so;
constructing a Precoder does, and fails loudly if it is not built.
"""
from .configs import CONFIGS, PAPER_POINTS, Config  # noqa: F401


def __getattr__(name):
    if name == "Precoder":
        from .api import Precoder
        return Precoder
    raise AttributeError(name)
