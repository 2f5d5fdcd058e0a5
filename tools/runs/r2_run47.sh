bash tools/ab_variants.sh 3 2 c32 c32g16 2>&1 | grep -v "^{" 
bash tools/ab_variants.sh 4 1 c32 c32g16 2>&1 | grep -v "^{"
