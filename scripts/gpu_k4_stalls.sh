mkdir -p gpurun_out
for spec in "persist cogvideox-5b 4" "default cogvideox-5b 0" "persist hunyuanvideo-720p 4" "default hunyuanvideo-720p 0"; do
  set -- $spec
  if [ $1 = default ]; then unset MODDIT_LIB_OVERRIDE; else export MODDIT_LIB_OVERRIDE=_variants/$1/libmoddit.so; fi
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_ -s 1 -c 1 -o gpurun_out/st_$1_$2 -f python scripts/k4_run_kernel.py $2 $3 2 > gpurun_out/st_$1_$2.log 2>&1
  ncu -i gpurun_out/st_$1_$2.ncu-rep --page source --csv > gpurun_out/st_$1_$2_source.csv 2>/dev/null
  rm -f gpurun_out/st_$1_$2.ncu-rep
done
