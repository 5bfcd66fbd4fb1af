import json,sys
for f in sys.argv[1:]:
    d=json.loads(open(f).read().strip().splitlines()[-1]); pk=d['per_kernel']
    print(f, 'ms/step',round(d['ms_per_step'],3), 'vcycle',round(d['vcycle_ms'],3), {k:round(v['ms']/v['launches']*1e3,1) for k,v in pk.items() if k.split('@')[0] in('prolong','restrict','residual','sweep') and k[-1] in '345'})
