bash tools/ab_variants.sh 3 2 s4 s2 g4 s3b 2>&1 | grep -v "^{" | cut -c1-260
bash tools/ab_variants.sh 4 1 s4 s2 g4 s3b 2>&1 | grep -v "^{" | cut -c1-260
