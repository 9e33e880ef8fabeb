for v in ${VARS:-base}; do
  if [ $v = base ]; then unset SDCSW_LIB_PATH; else export SDCSW_LIB_PATH=$PWD/build/var/$v.so; fi
  echo "== $v"; timeout 300 python tools/exp/synb_check.py ${TS:-511} 2>&1 | grep "bulk=1"
done
