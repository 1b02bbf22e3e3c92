for rep in 1 2; do
PMS8G_LIB=paper_1307_0571_b200/lib/libpms8g_base.so python scripts/branch50.py 4 | cut -c1-90 | sed 's/^/A /'
python scripts/branch50.py 4 | cut -c1-90 | sed 's/^/B /'
done
