mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; python3 -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print('value',round(d['value']),'ms',d['ms_per_step'],'e2e',round(d['e2e']['value']),d['e2e']['host_link_gbs'],d['e2e']['host_link_peak_gbs'],d['e2e']['host_link_frac'])
r=d['roofline']; print('dom',r['kernel'],round(r['frac'],3),'chain',round(r['chain_frac'],3))
for k in r['kernels']: print('  ',k['name'][:40],round(k['seconds']*1e6,1),round(k['frac'],3))
print('cpu',d['cpu_baseline'],'clocks',d['clocks'])
print(json.dumps(d['other_configs'],indent=1))
"
