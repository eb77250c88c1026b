"""Repro helper: the depth-order tests in file order, several rounds, in one process."""
import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import test_gpu_depth_ties as T
fails = 0
cases = [("short", T.test_short_runs_match_reference, ()), ("long", T.test_long_runs_match_reference, ()),
         ("equal", T.test_exactly_equal_depths_keep_source_order, ())]
cases += [(str(nf), T.test_depths_across_the_whole_near_far_range, nf) for nf in
          [(0.01, 100.0), (1e-3, 1e5), (0.5, 0.75), (2.0, 3.0e8), (1.0, 1.001), (4.0, 4.0005)]]
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    for name, fn, a in cases:
        try:
            fn(*a)
        except AssertionError as e:
            fails += 1
            print(it, name, "FAIL", [l for l in str(e).splitlines() if "Mismatch" in l])
print("fails", fails)
