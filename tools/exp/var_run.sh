cd $GRAFT_REPO_ROOT
for v in a b c; do
  echo "=== variant $v"
  SDCSW_LIB_PATH=build/var/r2$v.so python tools/exp/ring2_check.py 127 255 511 2>&1 | grep -v "rel per"
done
