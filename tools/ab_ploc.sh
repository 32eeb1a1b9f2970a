for v in default ${VARIANTS:-}; do
  if [ $v = default ]; then unset SBR_LIB_PATH; else export SBR_LIB_PATH=$PWD/paper_2504_21719_b200/_lib/variants/libsbr_$v.so; fi
  echo "== $v"; python tools/tree_quality.py 2>&1 | tail -2
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-cir --no-config5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('canyon', '%.3e'%d['value'], 'city c4', '%.3e'%d['config4']['value'])"
  python tools/vis_ab.py 2>&1 | tail -1 | cut -c1-140
done
