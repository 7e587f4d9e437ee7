"""Aggregate an ncu cuda,sass source export of bdf_tpc.cuh by function line ranges (plus whole other files)."""
import csv, sys, collections, bisect
csv.field_size_limit(1 << 30)
path = sys.argv[1]
ranges = [(109, 'tpc_factor'), (183, 'tpc_solve'), (218, 'coop_factor'), (254, 'nth_bit'), (292, 'wrms_reg'), (303, 'restore'), (323, 'restore_deferred'), (329, 'set_bdf'), (375, 'increase_bdf'), (404, 'decrease_bdf'), (426, 'order_deferred'), (458, 'adjust_order'), (464, 'set_eta'), (476, 'rescale'), (484, 'prepare_next'), (527, 'req_res'), (541, 'consume'), (624, 'hin_finish'), (633, 'start'), (650, 'setup_done'), (659, 'setup_decide'), (674, 'solve'), (714, 'nfail'), (736, 'errtest'), (828, 'step_top'), (852, 'attempt'), (967, 'store'), (1000, 'load'), (1051, 'ts_of'), (1055, 'ws_of'), (1057, 'lu_list'), (1063, 'trip')]
starts = [r[0] for r in ranges]
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
fname = None; hdr = None
with open(path, newline="") as f:
    for r in csv.reader(f):
        if not r: continue
        if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
        if r[0] == "Line No": hdr = r; continue
        if hdr is None: continue
        try: line = int(r[0])
        except ValueError: continue
        d = dict(zip(hdr, r))
        def num(k):
            try:
                return float(d.get(k, 0) or 0)
            except ValueError:
                return 0.0
        smp, ie, te = num("Warp Stall Sampling (All Samples)"), num("Instructions Executed"), num("Thread Instructions Executed")
        if fname == "bdf_tpc.cuh":
            i = bisect.bisect_right(starts, line) - 1
            key = "tpc:" + (ranges[i][1] if i >= 0 else "head")
        else:
            key = fname
        a = agg[key]; a[0] += smp; a[1] += ie; a[2] += te
ts = sum(a[0] for a in agg.values()) or 1; ti = sum(a[1] for a in agg.values()) or 1
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:34s} samples {100*a[0]/ts:5.1f}%  inst {100*a[1]/ti:5.1f}% ({a[1]:.3e})  thr/inst {a[2]/max(a[1],1):5.1f}")
