"""Phase timing of tile_pass_v3 (-DQT_V3_TIMING build libqtraj_v3t.so), CTA 7, on the
20-qubit depolarizing circuit of tools/v3_time.py (or C2 with --c2)."""
import ctypes, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads
from paper_2111_02396_b200 import qtraj
qtraj.LIB_PATH = qtraj.LIB_PATH.replace("libqtraj.so", "libqtraj_v3t.so")
ctx = qtraj.Context(0)
c = workloads.sycamore_grid_qcs(config=2) if "--c2" in sys.argv else workloads.random_circuit(20, depth=14, seed=9, max_arity=2, noise="depol", p=0.005)
plan = qtraj.Plan(qtraj.Circuit.from_description(c), max_fused=4, tile_bits=11)
state = torch.empty(384 << 20, dtype=torch.complex64, device="cuda")
out = ctx.run_trajectories(plan, state, seed=5, traj_count=768, batch=384, shots=1, observables=c.observables, profile=True)
buf = (ctypes.c_ulonglong * 32)()
qtraj.lib().qt_v3_timing_read(buf)
names = {0: "WG0 full wait", 1: "WG0 gather+split+st (TC)", 2: "WG0 MMA issue+wait", 3: "WG0 write back", 4: "WG0 CUDA-core gate",
         5: "WG0 item setup / misc", 6: "WG0 epilogues", 9: "WG0 item start (before wait)", 10: "loader empty wait", 11: "loader issue",
         12: "storer computed wait", 13: "storer store+lag"}
items = max(buf[14], 1)
print("WG0 items", buf[14], "pass_kernel_ms", out["stats"]["pass_kernel_ms"])
for k, nm in names.items():
    print(f"  {nm:32s} {buf[k]:14d} cyc  {buf[k] / items:9.0f} per WG0 item")
