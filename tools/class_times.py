"""Per-kernel-class average launch time (CUDA events per launch, eager mode) over a few
config-2 Schur solves: python tools/class_times.py [n s solves]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1312_5653_b200 as F  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
s = int(sys.argv[2]) if len(sys.argv) > 2 else 32
k = int(sys.argv[3]) if len(sys.argv) > 3 else 3
p = F.make_seeded_problem(n, 1e-4)
solver = F.SchurSolver(p, s, s, tol=1e-10, max_iter=2000)
solver.solve()
solver.profile(True)
solver.profile_read(reset=True)
for _ in range(k):
    solver.solve()
prof = solver.profile_read(reset=True)
tot = sum(v["ms"] for v in prof.values())
for c, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]):
    if v["launches"]:
        print(f"{c:14s} launches/solve {v['launches']/k:7.1f}  ms/solve {v['ms']/k:7.3f}  avg us {1000*v['ms']/v['launches']:8.2f}")
print(f"total ms/solve {tot/k:.3f}")
