# usage: bash tools/sass_ops.sh <function-name-regex>  -- opcode histogram of matching kernels in libsdp4.so
cuobjdump -sass paper_2410_15526_b200/libsdp4.so | awk -v pat="$1" '/Function :/ {keep = ($0 ~ pat)} keep && /\/\*[0-9a-f]+\*\// {for (i = 1; i <= NF; i++) if ($i ~ /^[A-Z][A-Z0-9_]+(\.|$)/) {split($i, a, "."); print a[1]; break}}' | sort | uniq -c | sort -rn | head -${2:-15}
