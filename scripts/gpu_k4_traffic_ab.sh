# DRAM bytes + duration of the K4 launch (ncu, cold caches) and warm CUDA-event time for library variants
#   VARIANTS="nopf2" bash scripts/gpu_k4_traffic_ab.sh
for v in default ${VARIANTS}; do
  if [ $v = default ]; then unset MODDIT_LIB_OVERRIDE; else export MODDIT_LIB_OVERRIDE=_variants/$v/libmoddit.so; fi
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:attn_ -c 1 --csv python scripts/k4_run.py ${CFG:-hunyuanvideo-720p} default 1 2>/dev/null | grep -E "dram__bytes|duration" | awk -F'","' -v v=$v '{print v, $(NF-2), $NF}'
done
VARIANTS="$VARIANTS" R=2 CFGS=${CFGS:-hunyuanvideo-720p,wan2.1-14b-720p} bash scripts/gpu_k4_variant_ab.sh
