# A/B of in-tree library variants (tools/build_variant.sh) on the 1M iteration: AB_VARIANTS="a b" bash tools/ab_variants.sh
cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in $AB_VARIANTS; do FGA_LIB_PATH=$PWD/paper_2009_14005_b200/_lib/libfga_$v.so python tools/iter_timing.py 20 2>&1 | tail -1; done; done
