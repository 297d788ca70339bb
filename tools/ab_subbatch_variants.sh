set -x
for v in "CPH_SUB_CHUNK=1" "CPH_SUB_CHUNK=5" "CPH_SUB_CHUNK=0" "CPH_SUB_CHUNK=1 CPH_SUB_STAGGER_US=400" "CPH_SUB_CHUNK=0 CPH_SUB_STAGGER_US=400"; do
  echo "== $v"; env $v timeout 300 python tools/ab_subbatch.py 4:21 2:17 2:34 2>&1 | tail -3
done
echo "== small R"; timeout 300 python tools/ab_subbatch.py 4:4 2:4 4:2 2:2 1:8 2>&1 | tail -5
