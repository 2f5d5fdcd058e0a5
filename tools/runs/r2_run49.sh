bash tools/ab_variants.sh 3 2 b10a b10b b8c b8d 2>&1 | grep -v "^{" 
