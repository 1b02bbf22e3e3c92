for v in ${VARIANTS:-base v12}; do
  if [ "$v" != base ]; then export PMS8G_LIB=$PWD/paper_1307_0571_b200/lib/$v/libpms8g.so; else unset PMS8G_LIB; fi
  echo "== variant $v"
  python scripts/profile_run.py 17 6 3 3 | head -1
  python scripts/profile_run.py 21 8 4 2 | head -1
  python scripts/profile_run.py 13 4 2 3 | head -1
done
