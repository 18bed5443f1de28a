"""cProfile of 50 inflate_edge calls (7-DOF bench region): where the Python wrapper spends its time."""
import sys, time, cProfile, pstats
sys.path.insert(0, '/root/repo')
from paper_2504_10783_b200 import fixtures as fx
from paper_2504_10783_b200.eizo import InflationParams, Segment, inflate_edge
from paper_2504_10783_b200.polytope import HPolytope
w = fx.franka7_world(); v1, v2 = fx.random_free_segment(w, seed=3)
dom = HPolytope.from_bounds(w.lower, w.upper); p = InflationParams(**fx.FRANKA_PARAMS); ck = w.checker()
for _ in range(5): inflate_edge(Segment(v1, v2), dom, p, ck, seed=7)
pr = cProfile.Profile(); pr.enable()
for _ in range(50): inflate_edge(Segment(v1, v2), dom, p, ck, seed=7)
pr.disable()
st = pstats.Stats(pr); st.sort_stats('tottime').print_stats(12)
