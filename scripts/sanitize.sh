for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"
  compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py 2>&1 | grep -vE "^ok|^skip" | tail -4
done
