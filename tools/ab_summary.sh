# print ms/step, fwd, adj, frac for ab logs matching TAG
for f in gpurun_out/ab_$1_*.log; do python -c "
import json,sys
env=open('$f').read().strip().splitlines()[-1]
for l in open('$f'):
    if l.startswith('{'):
        d=json.loads(l); r=d['roofline']; print('%-40s step %.3f fwd %.3f adj %.3f frac %.4f' % (env, d['ms_per_step'], r['t_fwd_ms'], r['t_adj_ms'], r['frac']))
"; done
tail -1 gpurun_out/pytest_gpu_$1.log
