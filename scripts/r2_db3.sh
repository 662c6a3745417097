set -u
python -m paper_1203_2739_b200.build > /dev/null
echo "== c3 4 panel_rows 16384"; timeout 300 python scripts/db_debug.py c3 4 16384 2>&1 | grep -v "^   rank\|^rank" | tail -8
echo "== c3 4 default"; timeout 300 python scripts/db_debug.py c3 4 2>&1 | grep -v "^   rank\|^rank" | tail -8
echo "== _c3w8 8"; timeout 300 python scripts/db_debug.py _c3w8 8 2>&1 | grep -v "^   rank\|^rank" | tail -8
echo "== c3 2"; timeout 300 python scripts/db_debug.py c3 2 2>&1 | grep -v "^   rank\|^rank" | tail -8
