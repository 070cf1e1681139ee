"""bench.sharded_bench at world 1 (NCCL, one GPU): exercises every sharded case
(configs 1-4) end to end; efficiency is ~1 by construction."""
import os, sys, json
sys.path.insert(0, os.getcwd())
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533", RANK="0", WORLD_SIZE="1")
import torch, torch.distributed as dist
torch.cuda.set_device(0)
dist.init_process_group("nccl")
import bench, paper_2310_05218_b200 as sc
print(json.dumps(bench.sharded_bench(torch, sc, 0, 1, 6548.0)))
dist.destroy_process_group()
