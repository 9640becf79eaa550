"""Time geer_loss at 1080p (CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_24053_b200 import train
a = torch.rand((1080, 1920, 3), device="cuda"); b = (a + 0.05 * torch.randn_like(a)).clamp(0, 1)
ws = train.LossWorkspace(); g = torch.empty_like(a)
for _ in range(3): train.loss_device(a, b, grad=g, workspace=ws)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): train.loss_device(a, b, grad=g, workspace=ws)
e1.record(); torch.cuda.synchronize(); print("geer_loss 1080p ms", e0.elapsed_time(e1) / 20)
