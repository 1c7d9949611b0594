cd $GRAFT_REPO_ROOT
python tools/build_variant.py count -- -DDENSE_COUNT > /dev/null 2>&1 || true
SFB_LIB=$GRAFT_REPO_ROOT/variants/count.so timeout 500 python tools/dense_count.py cfg4
./tools/micro/dmma_rate
