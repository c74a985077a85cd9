for r in 1 2; do
timeout 300 python scripts/k4_ab.py cogvideox-5b,hunyuanvideo-720p,wan2.1-14b-720p default 20 | sed "s/^/pf $r /"
MODDIT_LIB_OVERRIDE=_variants/nopf/libmoddit.so timeout 300 python scripts/k4_ab.py cogvideox-5b,hunyuanvideo-720p,wan2.1-14b-720p default 20 | sed "s/^/nopf $r /"
done
timeout 200 python scripts/k4_lsweep.py cogvideox-5b default 1,4,17 | sed "s/^/pf /"
MODDIT_LIB_OVERRIDE=_variants/nopf/libmoddit.so timeout 200 python scripts/k4_lsweep.py cogvideox-5b default 1,4,17 | sed "s/^/nopf /"
