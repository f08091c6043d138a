# Instruction count of a kernel's SASS: bash tools/sass_count.sh <.so/.o> <mangled-name-substring>
cuobjdump -sass "$1" | awk -v pat="$2" '/Function :/ {p = index($0, pat) > 0} p && /\/\*[0-9a-f]+\*\// {n++} END {print n}'
