"""kernel times (plain launches, events) of the 10.26M square (SURVEY config 5,
one part) unlinked vs self-linked: k_tile<LINK> and the exchange vs finalize"""
import sys
sys.path.insert(0, '/root/repo')
sys.path.insert(0, '.')
from paper_1807_00672_b200 import api, dist  # noqa: E402

sc = api.make_scenario("weak_square", weak_nx=2265)
part = dist.partition_raw(sc.raw, 1)
D = api.DeviceSolver
for link in (False, True):
    s = dist.LinkedPart(dist.rank_mesh(sc.raw, sc.bed, sc.manning, part, 0))
    s.info = lambda s=s: D.info(s)
    if link:
        dist.link_local([s])
    s.set_state(sc.state)
    s.advance(1e300, max_steps=20)
    D.set_profiling(s, True)
    D.advance_n_async(s, 50, t_end=1e300)
    D.synchronize(s)
    kt = D.kernel_times(s)
    D.set_profiling(s, False)
    print("linked" if link else "unlinked",
          {a: (round(b[0] / max(1, b[1]) * 1e3, 2), b[1]) for a, b in kt.items()})
    s.close()
