bash tools/ab_variants.sh 3 2 st4 st16 st32 2>&1 | grep -v "^{" | cut -c1-260
bash tools/ab_variants.sh 4 1 st4 st16 st32 2>&1 | grep -v "^{" | cut -c1-260
