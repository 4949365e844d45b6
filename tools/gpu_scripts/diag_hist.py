import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'tests/golden'); sys.path.insert(0,'.')
import numpy as np, refcpu, make_golden, paper_2101_11649_b200 as mx
for cid in ["mfd_6x5x4_mgr_pi","mfd_6x5x4_mgr_p","blocksys_unknown_amg","sdd60_two_field"]:
    case=[c for c in make_golden.CASES if c["id"]==cid][0]
    ptr, col, val, fields, labels, um, rhs = make_golden.build_problem(case["problem"])
    text = make_golden.strategy_text(case["strategy"])
    R = refcpu.RefHierarchy(ptr, col, val, fields, labels, text, um)
    H = mx.Hierarchy(mx.Matrix(ptr, col, val), mx.DofPartition(fields, labels), text, um)
    out={}
    for o in ["canonical","sequential"]:
        refcpu.set_dot_order(o); _, rr = R.solve(rhs, restart=30, max_iters=500, rel_tol=case["rtol"]); out["ref_"+o]=rr["history"]
    refcpu.set_dot_order("canonical")
    for o in ["mgs","cgs2"]:
        _, rep = H.solve(rhs, cfg=mx.KrylovConfig(restart=30, max_iters=500, rel_tol=case["rtol"], ortho=o)); out[o]=rep.residual_history
    print(cid, "n", ptr.size-1)
    for k,v in out.items(): print("  %-15s"%k, " ".join("%.17e"%x for x in v[:4]))
