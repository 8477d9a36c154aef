"""B200-native retrieval hot path of Teola (arXiv 2407.00326).

Vector search (fused inner-product scan + top-k), rerank scoring, top-k merge and corpus
normalisation as sm_100a kernels behind a C ABI (include/tsv.h), plus the host-side mirror
of the reference's primitive executor interface that dispatches to them.
"""

__version__ = "0.1.0"
