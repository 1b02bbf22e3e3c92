for v in vhead base; do
  if [ "$v" != base ]; then export PMS8G_LIB=$PWD/paper_1307_0571_b200/lib/$v/libpms8g.so; else unset PMS8G_LIB; fi
  echo "== $v"; python scripts/profile_run.py 17 6 0 3 | grep -E "wall"; SHARD=0/8 python scripts/profile_run.py 17 6 0 3 | grep -E "wall"; SHARD=0/8 python scripts/profile_run.py 21 8 0 2 | grep -E "wall"
done
unset PMS8G_LIB
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
