import sys, numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from test_gpu_cir import build
from test_oracle_cir import oracle_case
from paper_2504_21719_b200 import cir, _abi
name = sys.argv[1] if len(sys.argv) > 1 else "cfg1_default"
scene, _, cfg, txs, rxs = build(name)
osc, ocfg, otx, orx = oracle_case(name)
targets = np.array([r.position for r in rxs]); src = txs[0].position
scene.bind_frequency(cfg.frequency); scene.wedges
R = cir._sweep_rows(scene, src, targets, cfg, 0, cfg.num_samples)
g = {"key": R.key.cpu().numpy(), "pr": R.pr[:R.n].cpu().numpy(), "pf": R.pf[:R.n].cpu().numpy(),
     "chain": R.chain[:R.n].cpu().numpy()}
orows, oc = osc.cir_rows(src, targets, ocfg, 0, cfg.num_samples)
def canon(d):
    o = np.argsort(d["key"], kind="stable")
    return {k: v[o] for k, v in d.items()}
a, b = canon(g), canon(orows)
print("rows gpu", len(a["key"]), "oracle", len(b["key"]))
if len(a["key"]) == len(b["key"]):
    for k in a: print(k, "equal", np.array_equal(a[k], b[k]))
    bad = np.nonzero((a["pr"] != b["pr"]) | (a["key"] != b["key"]))[0][:5]
    for i in bad: print("diff", i, a["key"][i] >> 60, (a["key"][i] >> 20) & ((1<<40)-1), a["key"][i] & 0xfffff, b["key"][i] >> 60, (b["key"][i] >> 20) & ((1<<40)-1))
else:
    sa = set(a["key"].tolist()); sb = set(b["key"].tolist())
    for k in sorted(sa ^ sb)[:10]: print("only", "gpu" if k in sa else "orc", k >> 60, (k >> 20) & ((1<<40)-1), k & 0xfffff)
rr_o, co = osc.cir_select(src, targets, ocfg, g)
sel = torch.zeros(len(_abi.CIR_COUNTERS), dtype=torch.int64, device="cuda")
rr_g, n = cir._select_rows(R.params, R.key, R.pr, R.pf, R.chain, R.n, R.los_vis, cfg, sel, "cuda")
rr_g = rr_g[:n].cpu().numpy()
kg = np.where(rr_g >= 0, g["key"][np.maximum(rr_g, 0)], rr_g)
ko = np.where(rr_o >= 0, g["key"][np.maximum(rr_o, 0)], rr_o)
print("select on GPU rows: gpu", len(kg), "oracle", len(ko), "equal", np.array_equal(kg, ko))
if len(kg) == len(ko):
    d = np.nonzero(kg != ko)[0][:5]
    for i in d: print(i, kg[i] >> 60, (kg[i] >> 20) & ((1<<40)-1), ko[i] >> 60, (ko[i] >> 20) & ((1<<40)-1))
i = 14812
print("gpu", a["key"][i], a["pr"][i], a["pf"][i], a["chain"][i])
print("orc", b["key"][i], b["pr"][i], b["pf"][i], b["chain"][i])
print("w_hr equal", np.array_equal(scene._wedge_host["hash_r"], osc._w["hr"]), "wedges", len(scene.wedges), len(osc.wedges))
for gsmp in (9904,):
    R1 = cir._sweep_rows(scene, src, targets, cfg, gsmp, gsmp + 1)
    print("single gpu rows", R1.key[:R1.n].cpu().numpy(), R1.pr[:R1.n].cpu().numpy(), R1.chain[:R1.n].cpu().numpy())
    r1, _ = osc.cir_rows(src, targets, ocfg, gsmp, gsmp + 1)
    print("single orc rows", r1["key"], r1["pr"], r1["chain"])
