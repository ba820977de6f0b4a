"""oracle — float64 CPU reference of the HydraGNN training step (TEST INFRASTRUCTURE).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package. See hgnn_oracle.py for the citations
and the list of pins.
"""
from .hgnn_oracle import *  # noqa: F401,F403
from .hgnn_oracle import (adamw_step, allreduce_mean, backward, conv_forward,  # noqa: F401
                          degree_stat, forward, init_params, pack, param_specs, replay, scalers, shard,
                          splitmix64, train_step, zero_state)
