# stage release: after the stage's own DMMAs with a proxy fence (abtest/t_fence) vs deferred to the
# next iteration's full-wait (this tree); race check first, then same-box A/B
python tools/race_check.py 12 16384 U | tail -1
python tools/race_check.py 6 8192 L | tail -1
python tools/ab_trees.py abtest/t_fence . n16384 3
python tools/ab_trees.py abtest/t_fence . trtri 2
