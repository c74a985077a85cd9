mkdir -p gpurun_out
for rep in 1 2; do for v in ${VARIANTS:-v1 v5}; do MODDIT_LIB_OVERRIDE=_variants/$v/libmoddit.so MOD_ATTN_DEBUG=${DBG:-0} timeout 100 python scripts/attn_micro.py $1; done; done 2>&1 | grep -v Warn | tee gpurun_out/ab.log
