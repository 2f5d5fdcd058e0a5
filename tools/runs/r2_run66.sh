bash tools/ab_variants.sh 3 2 g4 g2 2>&1 | grep -v "^{" | cut -c1-260
bash tools/ab_variants.sh 4 1 g4 g2 2>&1 | grep -v "^{" | cut -c1-260
