for cfg in "17 6 3 2" "21 8 4 1 2"; do
  python scripts/profile_run.py $cfg | head -2
  PMS8G_NATURAL_ORDER=1 python scripts/profile_run.py $cfg | head -2
done
