cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
show() { python -c "
import json,sys
d=json.loads(open('$1').read().strip().splitlines()[-1])
print('BS', d['value'], d['ms_per_step'], 'c1', d['c1_1M_options'].get('ms_per_step'), 'gs', d['gpusession'].get('value'))
for k,v in d['workloads'].items(): print(' ', k, v['fused_iter_s'], v['unfused_iter_s'], v['dominant'])
"; }
for i in 1 2; do
timeout 900 python bench.py > gpurun_out/b59_$i.json 2>/dev/null; echo "default $i"; show gpurun_out/b59_$i.json
DK_VA_POOL_GB=0 timeout 900 python bench.py > gpurun_out/b59p_$i.json 2>/dev/null; echo "nopool $i"; show gpurun_out/b59p_$i.json
done
