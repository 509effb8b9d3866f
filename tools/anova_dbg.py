import sys; sys.path.insert(0,'.'); sys.path.insert(0,'oracle')
import numpy as np, workloads, pyoracle
import paper_2505_00448_b200 as ps
cfg = workloads.config(4)
ma = ps.make_matrix(cfg["a"], "categorical", na_sentinel=workloads.SENTINEL)
mb = ps.make_matrix(cfg["b"], "continuous", na_sentinel=workloads.SENTINEL)
req = ps.TestRequest("anova", ("stat","p","partial_eta2"))
res = ps.run(req, ma, mb)
Fq = mb.n_features
for g in [0, 100, 199]:
    ref = pyoracle.compute("anova", ma, mb, wanted={"stat","p","partial_eta2"}, lo=g*Fq, hi=(g+1)*Fq)
    a, b = res["stat"][g], ref["stat"][g]
    m = ~np.isnan(b)
    rel = np.abs(a[m]-b[m])/np.maximum(np.abs(b[m]),1e-300)
    idx = np.argsort(rel)[::-1][:5]
    hs = np.nonzero(m)[0][idx]
    print("g", g, "k", ma.category_counts[g], [(int(h), float(b[h]), float(rel[i]), float(res["partial_eta2"][g,h])) for i,h in zip(idx,hs)])
