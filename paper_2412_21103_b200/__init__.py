"""B200-native Needleman-Wunsch hot path (arXiv 2412.21103): C-ABI library + binding.

The product is libnw_b200.so (include/nw.h); this package holds its CUDA/C++
sources (csrc/), the build recipe (build.py), the ctypes binding (nw.py) and the
multi-process helpers (dist.py).
"""
from .nw import (NW_OK, NW_E_INVAL, NW_E_ALPHABET, NW_E_OVERFLOW, NW_E_NOMEM, NW_E_CUDA,  # noqa: F401
                 NW_E_TRUNC, NW_E_STATE, NW_E_DEADLOCK, NW_E_COMM, OPTIONS,
                 NW_DIAG, batch_paths, NW_LEFT, NW_SCORE_ONLY, NW_TRACEBACK, NW_UP, Context, NWError,
                 Traceback, lib, nw_align_batch, nw_align_batch_dev, nw_align_pair,
                 nw_align_pair_dev, nw_batch_ops_offsets, nw_batch_partition, nw_dist_unique_id,
                 nw_cblock_recv_bytes, nw_cblock_ipc_export, nw_cblock_ipc_import, nw_score_only,
                 nw_score_only_cblock,
                 nw_score_only_cblock_rank_dev, nw_score_only_dev,
                 nw_traceback, nw_traceback_dev, Msa, nw_msa_center_star, nw_msa_center_star_dev,
                 nw_align_pair_percell, nw_align_pair_percell_dev, nw_align_pair_linear,
                 nw_cooptimal)

__all__ = ["Context", "NWError", "Traceback", "lib", "nw_score_only", "nw_score_only_dev",
           "nw_score_only_cblock", "nw_score_only_cblock_rank_dev", "nw_cblock_recv_bytes",
           "nw_cblock_ipc_export", "nw_cblock_ipc_import",
           "nw_align_pair", "nw_align_pair_dev", "nw_traceback", "nw_traceback_dev",
           "nw_align_batch", "nw_align_batch_dev", "nw_batch_ops_offsets", "nw_batch_partition",
           "nw_dist_unique_id", "NW_DIAG", "NW_UP",
           "NW_LEFT", "NW_SCORE_ONLY", "NW_TRACEBACK", "batch_paths", "Msa",
           "nw_msa_center_star", "nw_msa_center_star_dev", "nw_align_pair_percell",
           "nw_align_pair_percell_dev", "nw_align_pair_linear",
           "nw_cooptimal", "OPTIONS"]
