import json,sys
d=json.load(open(sys.argv[1]))
print('tik ms',round(d['ms_per_step'],4),'e2e ms',round(d['e2e']['ms_per_step'],3))
for s,v in d['stages'].items(): print('  ',s,round(v['avg_us'],1))
for k in ('tv','config3'):
    if k in d:
        print(k,'ms/iter',round(d[k]['ms_per_iter'],4))
        for s,v in d[k]['stages'].items(): print('  ',s,round(v['avg_us'],1),round(v.get('frac',0),3))
if 'fp32' in d:
    f=d['fp32']; print('fp32 tik',round(f['ms_per_solve'],4), {k:(round(v.get('ms_per_iter',0),4) if isinstance(v,dict) else v) for k,v in f.items() if k.startswith('tv')})
if 'config4' in d: print('cfg4 tik',d['config4']['tikhonov_ms'],'tv',d['config4']['tv_ms_per_iter'], {k:round(v) for k,v in d['config4'].get('tv_stages_us',{}).items()})
