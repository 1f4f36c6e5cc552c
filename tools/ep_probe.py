"""Where does the EP step's time go at N=1?  torch.profiler (CUPTI) kernel table
+ host-side timing of one ExpertParallelMoE.step on the given workload."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

from moe_inputs import CONFIGS, make_inputs

wl = sys.argv[1] if len(sys.argv) > 1 else "mixtral"
cfg = CONFIGS[wl]
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29541", RANK="0", WORLD_SIZE="1")
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
from paper_2601_05296_b200.ep import ExpertParallelMoE

inp = make_inputs(cfg.T, cfg.d, cfg.h, cfg.E, cfg.k, dtype=cfg.dtype, seed=0, device=dev)
ep = ExpertParallelMoE(cfg.E, cfg.k, False)
args = [inp[n] for n in ("x", "w_gate", "w1", "w2", "w3", "dy")]
for _ in range(3):
    ep.step(*args)
torch.cuda.synchronize()
t0 = time.perf_counter()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    ep.step(*args)
e1.record()
host = (time.perf_counter() - t0) / 3
torch.cuda.synchronize()
print(f"{wl}: device {e0.elapsed_time(e1) / 3:.3f} ms/step, host issue {host * 1e3:.3f} ms/step")
from torch.profiler import ProfilerActivity, profile

with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    ep.step(*args)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=60))
prof.export_chrome_trace("gpurun_out/ep_trace.json")
dist.destroy_process_group()
