for env in "RELAPACK_DAG=0" "RELAPACK_SPLITK=0" "RELAPACK_BULK_CTAS=0" "RELAPACK_GRAPHS=0" "RELAPACK_REBASE=0"; do
  echo "== $env"
  env $env python tools/race_check.py 6 16384 U 2>&1 | tail -1
done
