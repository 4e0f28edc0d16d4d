"""Run bench.hmult_c3_sharded under torchrun (any world size, one GPU per rank):
torchrun --nproc-per-node R --master-addr 127.0.0.1 tools/shard_check.py"""
import os, sys, json
sys.path.insert(0, os.getcwd())
import torch, torch.distributed as dist
import bench
from paper_1908_06972_b200 import ckks
rank = int(os.environ.get("RANK", 0)); world = int(os.environ.get("WORLD_SIZE", 1))
dev = torch.device("cuda", 0); torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
r = bench.hmult_c3_sharded(torch, ckks, dev, 10, world, rank)
print(json.dumps(r))
dist.destroy_process_group()
