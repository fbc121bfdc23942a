import sys; sys.path.insert(0, ".")
import paper_2202_13821_b200 as P
r = P.run_case(P.CaseConfig.named("tgv", 32), P.RunOptions(degree=2, record_interval=0.05))
recs = r.records
inc = [(b.t, b.Ek - a.Ek) for a, b in zip(recs, recs[1:]) if b.Ek > a.Ek + 1e-12]
print("n", len(recs), "steps", r.steps, "increases", inc[:10])
for x in recs[::20]: print(f"{x.t:.2f} Ek={x.Ek:.10f} epsEk={x.epsEk:.6e} epsZ={x.epsZeta:.6e}")
integral = sum(0.5 * (b.epsEk + a.epsEk) * (b.t - a.t) for a, b in zip(recs, recs[1:]))
print("integral", integral, "drop", recs[0].Ek - recs[-1].Ek)
