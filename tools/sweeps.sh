#!/bin/bash
# Measured A/B sweeps behind the defaults recorded in DESIGN.md §5 (run on a GPU box):
#   tools/sweeps.sh <name>   name: whatif | whatif_c3 | agg_ctas | sample_ctas | sets | early_agg | l2 | align | pdl
# Each line prints sample-half / train-half / pipelined ms per step (tools/overlap_probe.py) or the
# bench headline for the given setting.
set -u
probe() { timeout 600 python tools/overlap_probe.py 2>/dev/null | head -3 | tr '\n' ' '; }
bench_line() {
  timeout 600 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/sweep.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/sweep.json')); print(round(d['value']), round(d['ms_per_step'],4), round(d['e2e']['value']))"
}
mkdir -p gpurun_out
case "${1:-whatif}" in
  whatif)  # kernel families removed from the captured step (results discarded; timing only)
    for k in "" "hg_aggregate_fwd:0" "hg_gemm_tc:0" "hg_wgrad_tc" "hg_wgrad_tc:2" \
             "hg_aggregate_bwd_scatter,hg_aggregate_bwd_finish" "hg_sage_top_fused" "hg_sgd_fused" \
             "hg_aggregate_fwd:0,hg_gemm_tc:0,hg_wgrad_tc:2"; do
      HG_WHATIF_SKIP="$k" probe; echo " <- skip [$k]"; done ;;
  whatif_c3)  # the same for C3 (GCN 2-layer, F=602, H=256): wgrad call 1 is the bottom layer
    for k in "" "hg_aggregate_fwd:0" "hg_gemm_tc:0" "hg_wgrad_tc:1" "hg_wgrad_tc" \
             "hg_aggregate_bwd_scatter,hg_aggregate_bwd_finish" "hg_softmax_xent" "hg_sgd_fused"; do
      HG_PROBE_WORKLOAD=c3 HG_WHATIF_SKIP="$k" probe; echo " <- skip [$k]"; done ;;
  agg_ctas) for c in 8 6 4 3 2; do HG_AGG_CTAS_PER_SM=$c probe; echo " <- agg CTAs/SM $c"; done ;;
  sample_ctas) for c in 8 4 2 1; do HG_SAMPLE_CTAS_PER_SM=$c probe; echo " <- sample CTAs/SM $c"; done ;;
  sets) for c in 2 3 4; do HG_SETS=$c probe; echo " <- sample sets $c"; done ;;
  early_agg) for e in 1 0; do HG_EARLY_AGG=$e probe; echo " <- early bottom aggregation $e"; done ;;
  l2) for mb in 0 24 32 48 64 96; do echo -n "L2 window $mb MB: "; HG_L2_PERSIST_MB=$mb bench_line; done ;;
  align) for a in 4 8 32; do echo -n "feature row align $a: "; HG_FEAT_ALIGN=$a bench_line; done ;;
  pdl) for p in 0 1; do echo -n "PDL $p: "; HG_PDL=$p bench_line; done ;;
  *) echo "unknown sweep $1"; exit 2 ;;
esac
