for k in "" "hg_aggregate_fwd:0" "hg_gemm_tc:0" "hg_wgrad_tc" "hg_wgrad_tc:2" "hg_aggregate_bwd_scatter,hg_aggregate_bwd_finish" "hg_sage_top_fused" "hg_sgd_fused" "hg_aggregate_fwd:0,hg_gemm_tc:0,hg_wgrad_tc:2"; do
  HG_WHATIF_SKIP="$k" timeout 600 python tools/overlap_probe.py 2>/dev/null | head -3 | tr '\n' ' '; echo " <- skip [$k]"; done
