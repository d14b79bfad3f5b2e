# Session-5 step 3: persistent block-solve microbench (ring carried across bricks)
mkdir -p gpurun_out
for r in 1 2; do for nb in 4096 32768; do echo "== persist R=$r nb=$nb"; timeout 200 tools/gpu/bin/thomas_persist_r$r $nb | head -8; done; done > gpurun_out/s5c_persist.txt 2>&1
cat gpurun_out/s5c_persist.txt
