#!/bin/bash
# One-off box facts for DESIGN.md (device properties, host cores/RAM, topology).
set -x
nvidia-smi
nvidia-smi topo -m
nproc; lscpu | head -20; free -g
python -c "
import torch
p=torch.cuda.get_device_properties(0)
print(p)
print('L2', p.L2_cache_size, 'smem/block optin', getattr(p,'shared_memory_per_block_optin',None), 'sms', p.multi_processor_count)
print('free/total', torch.cuda.mem_get_info())
"
