"""paper_2506_20677_b200 — B200-native hot path of Adaptive Hybrid Sort (arXiv 2506.20677).

A thin Python binding over the C ABI of ``lib/libahs.so`` (include/ahs.h).  The
functions carry the C names (``ahs_features``, ``ahs_select``, ``ahs_sort``,
``ahs_sort_host``); they only marshal torch tensors / numpy arrays into
pointers and sizes.  Every step of the path runs in the library's CUDA kernels;
there is no CPU fallback: if the extension is missing or no sm_100 device is
present, calls raise.
"""
from ._lib import (  # noqa: F401
    AHS_COUNTING, AHS_RADIX, AHS_GENERAL, AHS_I32, AHS_U32, AHS_I64, AHS_U64, FLAG_K_SATURATED,
    STRATEGY_NAMES, RULE_NAMES, FLAG_NAMES, Features, Thresholds, AhsError,
    lib, lib_path, ahs_version, ahs_thresholds_default, ahs_thresholds_from_env, ahs_workspace_bytes, ahs_sort_tmp_bytes, ahs_sort_tmp_bytes_dtype,
    ahs_sort_passes, ahs_features, ahs_select, ahs_sort, ahs_sort_host, ahs_host_scratch_bytes,
    ahs_launch_count, ahs_entropy_sorted, ahs_set_skip_trivial, ahs_set_count_kv_single, ahs_set_bucket_local, ahs_sort_plan, ahs_sort_executed_passes, ahs_rank_mode, ahs_lane_order_ok, RANK_MASKED, RANK_ORDERED, ahs_kernel_names, ahs_profile_begin, ahs_profile_end, ahs_profile_read,
    Workspace, sort, Model, ahs_select_model, ahs_sort_segments, ALGO4_NAMES, AHS_EMODEL, AHS_EMODELVER,
)
