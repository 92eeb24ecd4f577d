# build the extension; exit 1 (printing the errors) unless it succeeded
out=$(python -m paper_1208_4772_b200.build --no-oracle 2>&1)
echo "$out" | grep -E "error" | head -5
echo "$out" | tail -1 | grep -q "^built" && echo built
