for e in 1 0; do HG_EARLY_AGG=$e timeout 600 python tools/overlap_probe.py 2>/dev/null | head -3 | tr '\n' ' '; echo " <- early agg $e"; done
HG_EARLY_AGG=0 HG_WHATIF_SKIP="hg_gemm_tc:0" timeout 600 python tools/overlap_probe.py 2>/dev/null | head -3 | tr '\n' ' '; echo " <- early agg 0, no bottom GEMM"
