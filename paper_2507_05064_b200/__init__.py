"""B200-native VIF (Vecchia-inducing-points full-scale) factor + Gaussian NLL, arXiv 2507.05064.

The product is libvif.so (csrc/, C ABI in include/vif.h); `vif` is its thin ctypes binding.
"""
from .vif import (EXPORTED, LIB_PATH, Terms, Theta, VifError, VifModel, load_library, owned_rows,  # noqa: F401
                  vif_copy_U, vif_create, vif_destroy, vif_factor, vif_last_error, vif_launch_count,
                  vif_nccl_unique_id, vif_nll, vif_partition, vif_profile, vif_set_data, vif_stage_name,
                  vif_stage_times, vif_workspace_bytes)

__all__ = ["VifModel", "Theta", "Terms", "VifError", "load_library"] + list(EXPORTED)
