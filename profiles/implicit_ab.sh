for v in ${VARIANTS:-base}; do
  if [ $v = base ]; then unset ST_VARIANT; else export ST_VARIANT=$v; fi
  python -c "
import sys; sys.argv=['bench.py']; sys.path.insert(0,'.')
import bench, json; r = bench.implicit_measure(0, cpu=False); print('$v', round(r['ms_per_be_step'],3), round(r['us_per_cg_iteration'],1), round(r['explicit_us_per_step'],2))"
done
