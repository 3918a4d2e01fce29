import sys; sys.path.insert(0,'.')
import paper_1508_05488_b200 as P
c=P.Context(0)
c.set_spa_path(P.SPA_SORT)
for d,n in (('circle',60000),('uniform_disk',200000),('gaussian',100000)):
    r=c.convex_hull(P.generate(d,n,1), P.PipelineConfig(chunk_count=7)); print(d, r.stats.n_hull, r.diag.spa_path)
c.set_spa_path(P.SPA_AUTO)
r=c.convex_hull(P.generate('circle',70000,2)); print('circle auto', r.stats.n_hull, r.diag.convex_fast_path)
