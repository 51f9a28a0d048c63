bash tools/gpu_variants.sh v2f "nocold16 nocold18 nocold20"
VARENV="DSMC_CAPW=416" bash tools/gpu_variants.sh v2f416 "nocold16 nocold18 nocold20"
VARENV="DSMC_CAPW=384" bash tools/gpu_variants.sh v2f384 "nocold20"
