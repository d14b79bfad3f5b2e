# quick.sh on the in-tree library, then bench-only A/B against the given variants
bash tools/gpu/quick.sh
bash tools/gpu/ab.sh "$@" | grep -E "^(base|$(echo "$@" | tr ' ' '|')) "
