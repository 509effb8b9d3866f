import sys; sys.path.insert(0, ".")
import numpy as np, bench, workloads
import paper_2505_00448_b200 as ps
cfg = workloads.config(bench.parse_config("2"))
a, b, ka, kb = bench.build_inputs(cfg, "spearman")
m = ps.make_matrix(a, ka, na_sentinel=workloads.SENTINEL)
res = ps.run(ps.TestRequest("spearman", ("p",)), m)
p = res["p"][np.triu_indices(res["p"].shape[0], 1)]
p = p[~np.isnan(p)]
bits = p.view(np.uint64)
hi = bits >> np.uint64(32)
u, inv, cnt = np.unique(hi, return_inverse=True, return_counts=True)
print("m", p.size, "distinct hi", u.size, "max run", cnt.max())
big = np.nonzero(cnt > 64)[0]
for g in big[:10]:
    sel = bits[inv == g]
    print("run hi=%x len %d distinct full %d  p~%r" % (u[g], cnt[g], np.unique(sel).size, p[inv == g][0]))
