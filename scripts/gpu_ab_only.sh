# A/B of exp/lib_*.so only (no tests): AB_TAG, AB_WL
bash scripts/gpu_ab.sh ${AB_TAG:-ab} ${AB_WL:-cfg3} > /dev/null 2>&1
for f in gpurun_out/${AB_TAG:-ab}_lib_*.json; do python -c "
import json,sys; j=json.loads(open('$f').read().strip().splitlines()[-1]); r=j['roofline']
print('$f'.split('/')[-1], round(j['value'],1), 'e2e', round(j['e2e']['value'],1), 'kernel', round(r['kernel_ms'],4), 'frac', round(r['frac'],3), 'slow', j.get('slow_path_items'))"; done
