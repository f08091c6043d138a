# Tile-shard per-rank times with and without the split tree, three scene seeds (experiments build).
export SRT_LIBSRT_PATH=paper_2504_06598_b200/libsrt_exp.so
for s in 0 1 2; do for C in 0 7; do echo "seed $s C=$C"; SRT_SPLIT_CELLS=$C timeout 300 python tools/shard_times.py $s 2>&1 | tail -4; done; done
