for v in "" at49d1727 at1661a23 at0f25bab; do
  for rep in 1 2; do
    r=$(BQG_LIB_VARIANT=$v timeout 600 python -m pytest tests/test_sharded.py -q -x -k "grouped_sharded" 2>&1 | tail -1)
    echo "variant '$v' rep $rep: $r"
  done
done
