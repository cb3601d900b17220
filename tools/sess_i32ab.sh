# A/B of int32-kernel library variants (tools/variants.py): VARIANTS="name=-DFLAG ..."
VARIANTS_PREBUILT=1 python tools/variants.py ${VARIANTS} > /dev/null 2>&1
for v in ${VARIANTS}; do
 v=${v%%=*}
 for a in "--force-group 2" "--force-group 8" "--force-group 2 --mode extend" "--force-group 8 --mode extend"; do
  SALOBA_LIB=build/variants/$v/libsaloba.so python bench.py --pairs 300000 --steps 3 --force-path 1 $a --no-cpu-baseline --e2e-steps 0 --start-steps 0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$v $a\", d[\"roofline\"][\"achieved\"])"
 done
 SALOBA_LIB=build/variants/$v/libsaloba.so python bench.py --config 4 --pairs 100000 --steps 2 --no-cpu-baseline --e2e-steps 0 --start-steps 0 --band 100 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$v band\", d[\"banded\"][\"gcups_band_cells\"])"
done
