# A/B of K4 library variants (_variants/NAME) on the bench workloads with scripts/k4_ab.py, alternating R rounds.
#   VARIANTS="tma3d" CFGS=hunyuanvideo-720p,wan2.1-14b-720p R=2 bash scripts/gpu_k4_variant_ab.sh
for r in $(seq 1 ${R:-2}); do
for v in default ${VARIANTS}; do
  if [ $v = default ]; then unset MODDIT_LIB_OVERRIDE; else export MODDIT_LIB_OVERRIDE=_variants/$v/libmoddit.so; fi
  timeout 300 python scripts/k4_ab.py ${CFGS:-hunyuanvideo-720p,wan2.1-14b-720p} ${KERNS:-default} ${REPS:-20} | sed "s/^/$v $r /"
done; done
