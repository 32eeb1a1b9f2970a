L=$PWD/paper_2504_21719_b200/_lib/variants
for v in default ge1 ge2 default ge1 ge2; do
  if [ $v = default ]; then unset SBR_LIB_PATH; else export SBR_LIB_PATH=$L/libsbr_$v.so; fi
  echo "$v $(timeout 300 python tools/vis_ab.py 2>&1 | tail -1)"
done
