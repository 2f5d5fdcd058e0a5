bash tools/ab_variants.sh 3 3 bpf0 2>&1 | grep -v "^{" 
bash tools/ab_variants.sh 4 2 bpf0 2>&1 | grep -v "^{"
