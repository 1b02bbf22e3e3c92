for v in ${VARIANTS:-base v12}; do
  if [ "$v" != base ]; then export PMS8G_LIB=$PWD/paper_1307_0571_b200/lib/$v/libpms8g.so; else unset PMS8G_LIB; fi
  echo "== variant $v"
  python scripts/profile_run.py 23 9 0 1 4 | head -1
  python scripts/profile_run.py 21 8 3 1 2 | head -1
  python scripts/profile_run.py 17 6 4 2 | head -1
done
