"""STP (synergistic tensor + pipeline parallel schedule, arXiv 2510.27257)
hot path on B200: C-ABI library libstp.so + thin Python binding.

Importing this package sets CUDA_DEVICE_MAX_CONNECTIONS=32 (if unset) so
that it takes effect before CUDA initialises: the executor drives up to
2 + 4 streams plus NCCL's own, and with the default 8 hardware work queues a
posted (spinning) NCCL recv can falsely serialise the matching send of the
same GPU (observed as a PP=2 deadlock).
"""
import os

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
