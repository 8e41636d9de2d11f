"""B200-native expert-parallel MoE layer of Lina (arXiv 2210.17223).

The compute lives in ``liblina.so`` (CUDA for sm_100a + NCCL) behind the C ABI of
``include/lina.h``; ``lina`` is its thin ctypes binding.  Importing this package
loads the library and fails loudly when it has not been built — there is no CPU
fallback.
"""
from . import lina  # noqa: F401
from .lina import (ABI_SYMBOLS, Comm, LinaError, MoELayer, PopProfile, lina_allreduce_submit,  # noqa: F401
                   lina_allreduce_wait, lina_comm_init, lina_get_unique_id, lina_moe_backward,
                   lina_moe_forward, lina_moe_infer_forward, lina_moe_infer_forward_two_phase,
                   lina_moe_infer_workspace_size,
                   lina_moe_workspace_size, lina_placement_compute, lina_profile_enable,
                   lina_phase_two_check, lina_profile_read, lina_replica_split,
                   lina_sched_config, lina_sched_stats, lina_version, load, make_desc,
                   lina_infer_last_rows, lina_pack_decide, lina_pack_weights, PackController)

load()
