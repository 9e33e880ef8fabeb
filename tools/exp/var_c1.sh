cd $GRAFT_REPO_ROOT
for v in ${VARS:-default p1 p2 p3 p4 p2t p0t}; do
  if [ $v = default ]; then python tools/exp/var_c1.py; else SDCSW_LIB_PATH=build/var/$v.so python tools/exp/var_c1.py; fi
done
