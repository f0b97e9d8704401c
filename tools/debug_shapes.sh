i=0
for n in $(seq 1 40); do
  python tools/debug_shapes.py $i; rc=$?
  if [ $rc -eq 0 ]; then break; fi
  i=$rc
done
