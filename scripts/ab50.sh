# A/B of two builds on (50,21) anchor 0 branches 0..15
A=${LIBA:-paper_1307_0571_b200/lib/libpms8g_base.so}
B=${LIBB:-paper_1307_0571_b200/lib/libpms8g.so}
for rep in 1 2; do
PMS8G_LIB=$A python scripts/branch50.py ${NB:-16} | cut -c1-100 | sed 's/^/A /'
PMS8G_LIB=$B python scripts/branch50.py ${NB:-16} | cut -c1-100 | sed 's/^/B /'
done
