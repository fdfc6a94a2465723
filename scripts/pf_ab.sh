cd $GRAFT_REPO_ROOT
for pf in 0 1 2 3; do LAQ_PREFETCH=$pf python - <<'PY'
import os,sys
sys.argv=['x']
exec(open('scripts/scan_ab.py').read().split('res = {}')[0])
import torch
for variant in ("direct",):
    plans = [ds.prepare(Q.spec_with_dial(Q.group_defs(gr)[qi], gr, d)) for (gr, qi), d in DIALS.items()]
    out=[]
    for p in plans:
        p.build_codes()
        for _ in range(3): p.scan()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): p.scan()
        e1.record(); torch.cuda.synchronize()
        out.append(round(e0.elapsed_time(e1)/20,4))
    print("pf", os.environ["LAQ_PREFETCH"], out, round(sum(out),4), flush=True)
PY
done
