for c in 8 4 2; do HG_AGG_CTAS_PER_SM=$c timeout 600 python tools/overlap_probe.py 2>/dev/null | head -3 | tr '\n' ' '; echo " <- agg ctas/SM $c"; done
HG_EARLY_AGG=0 timeout 600 python tools/overlap_probe.py 2>/dev/null | head -3 | tr '\n' ' '; echo " <- early off"
