for a in 4 32; do for f in 4 32; do HG_ACT_ALIGN=$a HG_FEAT_ALIGN=$f timeout 600 python tools/overlap_probe.py 2>/dev/null | head -3 | tr '\n' ' '; echo " <- act $a feat $f"; done; done
