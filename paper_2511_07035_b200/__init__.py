"""paper_2511_07035_b200 — B200-native GoCkpt hot path (arXiv 2511.07035).

The multi-step overlapped checkpoint: a fused sm_100a AdamW kernel that packs
one partition of the fp32 optimizer state plus the step's gradient prefix into
an HBM staging ring, a copy-engine (or zero-copy) drain into pinned host
memory on a side stream, and a gradient-assisted replay (host pool or GPU
kernel) that makes the assembled checkpoint equal the synchronous snapshot.
The compute lives in ``libgockpt.so`` behind the C ABI of ``include/gockpt.h``;
this package is the thin binding. There is no CPU fallback: importing the
binding without the built library raises.
"""

from .gockpt import (GoCkpt, HostCheckpoint, make_step_record, plan_parts, replay_host, replay_device,
                     adamw_step, h_generate, d2h_copy, checksum, device_count,
                     write_checkpoint, write_checkpoint_log, read_header, read_log_header, load_checkpoint,
                     load_checkpoint_range, recommend_k,
                     ring_bytes_required, GEN_MASTER, GEN_EXP_AVG, GEN_EXP_AVG_SQ, GEN_GRAD)
from ._lib import GckError, lib, LIB_PATH
from .optim import CheckpointedAdamW

__all__ = ["GoCkpt", "CheckpointedAdamW", "HostCheckpoint", "make_step_record", "plan_parts", "replay_host", "replay_device",
           "adamw_step", "h_generate", "d2h_copy", "checksum", "device_count",
           "write_checkpoint", "write_checkpoint_log", "read_header", "read_log_header", "load_checkpoint",
           "load_checkpoint_range", "recommend_k",
           "ring_bytes_required", "GckError", "lib", "LIB_PATH",
           "GEN_MASTER", "GEN_EXP_AVG", "GEN_EXP_AVG_SQ", "GEN_GRAD"]
