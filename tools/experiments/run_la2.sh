for la in 0 1; do echo "LA=$la"; RELAPACK_GETRF_LA=$la PYTHONPATH=. timeout 300 python tools/getrf_breakdown.py 16384; done
echo "LA=0 cluster16"; RELAPACK_GETF2_CLUSTER=16 PYTHONPATH=. timeout 300 python tools/getrf_breakdown.py 16384
