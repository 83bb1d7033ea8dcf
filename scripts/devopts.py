"""Development probes only: map TC_<OPTION>=value environment variables onto the library's
explicit schedule options (tc_set_option).  The product library itself never reads the
environment; this shim keeps the A/B shell scripts under scripts/gpu/ working."""
import os

NAMES = ("vmajor", "vzone_log2", "vlow_all", "vm_bias", "dense_factor", "hub_unroll", "l2_persist_mb",
         "l2_target", "concurrent", "share", "midwarp", "light", "skew", "light_vec", "shard_model",
         "shard_ovh", "shard_ucap", "dense_ranks", "bucket", "count_stats", "hubpack", "rank_primary",
         "shard_ovh2", "copy_threads", "seg_fork", "shard_w_dense", "shard_w_sparse", "shard_w_light",
         "shard_w_stage", "shard_w_edge", "shard_w_hub", "shard_w_vlow", "shard_w_vedge", "vin_overlap",
         "vin_grid", "seg_k16", "vhub", "seg_w2k", "vhub_unroll", "vhub_blocks", "vhub_b16w", "hub_cap_div", "vix")


def apply():
    from paper_1503_00576_b200 import _lib
    for name in NAMES:
        v = os.environ.get("TC_" + name.upper())
        if v is not None:
            _lib.set_option(name, int(v))
