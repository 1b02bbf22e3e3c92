for o in "" 1; do
echo "no_order=$o"
export PMS8G_NO_TASK_ORDER=$o; [ -z "$o" ] && unset PMS8G_NO_TASK_ORDER
SHARD=0/8 python scripts/profile_run.py 17 6 0 2 | grep -E "wall|idle"
python scripts/profile_run.py 17 6 0 2 | grep -E "wall|idle"
SHARD=0/8 python scripts/profile_run.py 21 8 0 2 | grep -E "wall|idle"
python scripts/profile_run.py 13 4 0 3 | grep -E "wall|idle"
done
unset PMS8G_NO_TASK_ORDER
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
