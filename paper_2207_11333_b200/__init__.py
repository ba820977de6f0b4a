"""paper_2207_11333_b200 — B200-native (sm_100a) HydraGNN PNA-GCNN data-parallel training step.

The compute path lives in ``lib/libhgnn.so`` (C-ABI: ``include/hgnn.h``;
sources in ``csrc/``). ``hgnn`` is the thin ctypes binding.
"""
from . import hgnn  # noqa: F401
from .hgnn import (Context, HgError, Store, hg_backward, hg_batch_offsets, hg_forward, hg_pack,  # noqa: F401
                   hg_pack_host, hg_param_layout, hg_params_init_host, hg_shard, hg_step, hg_train_step,
                   make_adamw, make_config, unpack_blob)

__all__ = ["hgnn", "Context", "Store", "HgError", "make_config", "make_adamw"]
