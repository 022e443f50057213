python tools/race_check.py 12 16384 U
RELAPACK_PDL=0 python tools/race_check.py 8 16384 U
