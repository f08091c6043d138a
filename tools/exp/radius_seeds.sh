# PLOC radius vs scene seed (is the radius effect tree quality or luck?), 1M SH-3, 1080p, 1 spp
for seed in 0 1 2; do for r in 8 12 16 20 24 32; do
  echo -n "seed $seed radius $r: "
  SRT_SEED=$seed SRT_PLOC_RADIUS=$r python tools/time_frames.py 1000000 1920 1080 1 1 9 | grep -o "build [0-9.]* ms\|trace [0-9.]* ms" | tr '\n' ' '; echo
done; done
