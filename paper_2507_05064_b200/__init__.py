"""B200-native VIF (Vecchia-inducing-points full-scale) factor + Gaussian NLL, arXiv 2507.05064.

The product is libvif.so (csrc/, C ABI in include/vif.h); `vif` is its thin ctypes binding.
"""
from .vif import (EXPORTED, LA_OPS, LIB_PATH, LaOpts, LaTerms, Terms, Theta, VifError, VifModel,  # noqa: F401
                  load_library, owned_rows, vif_copy_U, vif_create, vif_destroy, vif_factor, vif_grad,
                  vif_gram, vif_grad_workspace_bytes, vif_la_apply, vif_la_nll, vif_la_prepare, vif_la_workspace_bytes,
                  vif_last_error, vif_launch_count, vif_nccl_unique_id, vif_neighbors, vif_nll, vif_owned_rows,
                  vif_partition, vif_predict, vif_predict_workspace_bytes, vif_profile, vif_set_data,
                  vif_stage_data, vif_stage_name, vif_stage_times, vif_workspace_bytes)

__all__ = ["VifModel", "Theta", "Terms", "VifError", "LaOpts", "LaTerms", "load_library"] + list(EXPORTED)
