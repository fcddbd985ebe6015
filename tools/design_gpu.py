"""Time the GPU designer on the shipped designs' configurations (DesignConfig():
4 restarts + the zero start, up to 2000 sweeps each) and compare the objective
with the shipped file (which the reference's designer produced).
Usage: python tools/design_gpu.py [name ...]   (default: the N=16/32 designs)"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2505_23618_b200 import designer as G, matio  # noqa: E402
from paper_2505_23618_b200.transforms import build_transform  # noqa: E402

names = sys.argv[1:] or ["sub8_post_dct2_dst7_n16", "band4_pre_dst3_dst7_n16",
                         "band6_pre_dst3_dst7_n16", "sub8_post_dct2_dst7_n32",
                         "band6_pre_dst3_dst7_n32", "band6_pre_dst3_dst7_n64"]
for name in names:
    ref = matio.load_designed(name)
    n = ref.pattern.size
    b, d = build_transform(ref.base, n), build_transform(ref.target, n)
    t0 = time.perf_counter()
    adj = G.optimize_adjustment(b, d, ref.pattern, ref.side, G.DesignConfig())
    dt = time.perf_counter() - t0
    h = b.entries @ ref.realized if ref.side.value == "pre" else ref.realized @ b.entries
    ref_obj = G.weighted_error(h, d.entries, G.default_alpha(n))
    rel = (adj.objective - ref_obj) / ref_obj
    print(f"{name}: {dt:.2f} s on the GPU, objective {adj.objective:.12g} vs shipped "
          f"{ref_obj:.12g} (rel {rel:+.2e}), restart {adj.restart_index}, "
          f"sweeps {len(adj.objective_trace) - 1}, converged {adj.converged}", flush=True)
