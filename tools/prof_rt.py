"""Fused round trip (dctadj_roundtrip_2d) on config-2-shaped batches: per-launch
time for the current DCTADJ_RT_VARIANT, sub-block post (DCT-8) and band-6 pre
(DST-7).  Usage: python tools/prof_rt.py [iters]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2505_23618_b200 import matio, pipeline  # noqa: E402
from paper_2505_23618_b200.design import dct8_adjustment_from_dst7  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 50
x = torch.randn(65536, 32, 32, device="cuda") * 24
for name, adj in (("sub8 post dct8", dct8_adjustment_from_dst7(matio.load_designed("sub8_post_dct2_dst7_n32"))),
                  ("band6 pre dst7", matio.load_designed("band6_pre_dst3_dst7_n32"))):
    t = pipeline.make_adjusted_transform(adj)
    pipeline.roundtrip_adjusted_2d(t, t, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        pipeline.roundtrip_adjusted_2d(t, t, x)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / iters * 1e3
    print(f"{name}: {us:.1f} us per round trip, {805306368 / us / 1e3:.0f} GB/s algorithmic")
