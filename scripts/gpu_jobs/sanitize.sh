timeout 600 compute-sanitizer --tool memcheck --show-backtrace device python scripts/probe_vcycle.py full_64 64 1 2>&1 | head -60
