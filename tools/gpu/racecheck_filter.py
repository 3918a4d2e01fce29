"""Inputs for compute-sanitizer racecheck/synccheck over the default
(pre-filtered) path, its deferred chunk variant and the overflow hand-over."""
import sys; sys.path.insert(0, '.')
import paper_1508_05488_b200 as P
c = P.Context(0)
for d, n in (('uniform_square', 300000), ('uniform_disk', 200000), ('gaussian', 200000),
             ('duplicates_heavy', 50000)):
    r = c.convex_hull(P.generate(d, n, 1)); print(d, r.stats.n_hull, r.diag.spa_path)
c.set_spa_path(P.SPA_FILTER_SORTED)
r = c.convex_hull(P.generate('uniform_square', 300000, 2)); print('filter_sorted', r.stats.n_hull)
c.set_spa_path(P.SPA_FILTER)
r = c.convex_hull(P.generate('circle', 400000, 3)); print('circle filter', r.stats.n_hull, r.diag.spa_path)
