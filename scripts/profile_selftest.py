"""Host vs device time of the reference CLI selftest on the B200 backend (cProfile)."""
import cProfile, io, os, pstats, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "baseline", "_ref")]
import hebnn.cli as cli
from paper_1806_03461_b200.backend import TfheContext
cli.SimContext = TfheContext
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
rc = cli.main(["selftest"])
pr.disable()
print("rc", rc, "wall", time.perf_counter() - t0)
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(35)
print(s.getvalue())
