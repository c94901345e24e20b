for mb in 0 24 48 64 96; do HG_L2_PERSIST_MB=$mb timeout 600 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/b_l2_$mb.json 2>/dev/null; echo "mb=$mb"; python -c "
import json; d=json.load(open('gpurun_out/b_l2_$mb.json')); r=d['roofline']; print(round(d['value']), round(d['ms_per_step'],4), round(r['avg_launch_ms']*1000,1), round(r['frac'],3), round(d['e2e']['value']))"; done
python -c "
import torch, sys; sys.path.insert(0,'.')
from paper_2311_13225_b200 import _lib
print('persist max', _lib.load().hg_l2_persist_max())"
