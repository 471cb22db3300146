import os, sys
os.environ["NCCL_DEBUG"] = "INFO"
import torch, torch.distributed as dist
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
x = torch.ones(4, device="cuda"); y = torch.empty(4, device="cuda")
dist.reduce_scatter_tensor(y, x); torch.cuda.synchronize()
print("probe ok", y.tolist(), torch.cuda.nccl.version(), file=sys.stderr)
dist.destroy_process_group()
