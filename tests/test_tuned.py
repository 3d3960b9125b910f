"""tuned.json (tools/tune.py's measured plans) against the kernels' plan tables (CPU): every entry names a
plan the library instantiates and whose footprint fits; Grid() applies an entry only to exactly that kind
and shape with the plan left to the library."""
import paper_1410_3060_b200 as st
from paper_1410_3060_b200 import model


def test_tuned_entries_are_instantiated_fitting_plans():
    import json
    import os
    d = json.load(open(os.path.join(os.path.dirname(st.LIB_PATH), "tuned.json")))
    assert d
    for key, plan in d.items():
        kind = int(key.split(":")[0])
        if plan["variant"] == st.ST_VARIANT_COOP:
            continue
        if kind == model.K25V and plan["bt"] == 2:
            cfgs = {c[0]: c[1:] for c in model.pipe25_plans()}
            assert plan["tile_cfg"] in cfgs
            assert model.pipe25_footprint(*cfgs[plan["tile_cfg"]])["fits"]
        else:
            cands = [(cfg, a) for k, bt, cfg, a in model.pipe_plans() if k == kind and bt == plan["bt"]]
            assert any(cfg == plan["tile_cfg"] for cfg, _ in cands), (key, plan)
            a = dict(cands)[plan["tile_cfg"]]
            assert model.pipe_footprint(kind, plan["bt"], **a)["fits"]


def test_tuned_plan_lookup_is_exact():
    assert st.tuned_plan(st.ST_7PT_VAR, 512, 512, 512)["bt"] >= 1
    assert st.tuned_plan(st.ST_7PT_VAR, 512, 512, 511) is None
