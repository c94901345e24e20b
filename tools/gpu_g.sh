for c in 8 4 2 1; do HG_SAMPLE_CTAS_PER_SM=$c timeout 600 python tools/overlap_probe.py 2>/dev/null | head -3 | tr '\n' ' '; echo " <- ctas/SM $c"; done
