timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_pdl.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_pdl.log
for p in 0 1; do HG_PDL=$p timeout 600 python bench.py --no-cpu-baseline --phases > gpurun_out/b_pdl_$p.json 2>/dev/null; echo "pdl=$p"; python -c "
import json; d=json.load(open('gpurun_out/b_pdl_$p.json')); print(round(d['value']), round(d['ms_per_step'],4), round(d['e2e']['value']), {k: round(v*1000,1) for k,v in d['phases_ms'].items()})"; done
HG_PDL=1 timeout 600 python tools/overlap_probe.py 2>/dev/null | head -3
