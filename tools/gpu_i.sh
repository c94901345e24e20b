for a in 4 8 32; do HG_FEAT_ALIGN=$a timeout 600 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/b_al_$a.json 2>/dev/null; echo "align=$a"; python -c "
import json; d=json.load(open('gpurun_out/b_al_$a.json')); r=d['roofline']; print(round(d['value']), round(d['ms_per_step'],4), round(r['avg_launch_ms']*1000,1), round(r['frac'],3), round(d['e2e']['value']))"; done
