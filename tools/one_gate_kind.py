"""Single blocked-kernel launch for profiling: n=21, 640 CU3 gates on qubit
pairs (q, q+1) with q cycling over 0..4 (one pass per 48 gates)."""
import sys
sys.path.insert(0, "/root/repo/tools")
sys.path.insert(0, "/root/repo")
from pass_cost import measure
n = int(sys.argv[1]) if len(sys.argv) > 1 else 21
lo = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ms, passes, gates = measure(n, [(lo + i % 5, lo + i % 5 + 1) for i in range(640)], reps=1)
print(f"n={n} lo={lo}: {ms:.3f} ms, {passes} passes, {1e3 * ms / gates:.3f} us/gate")
