timeout 600 python scripts/time_libs.py --frames 1 --scene c4 variants/*.so 2>&1 | tail -3
timeout 600 python scripts/time_libs.py --frames 1 --scene c4 --fb 0 variants/*.so 2>&1 | tail -3
timeout 600 python scripts/time_libs.py --frames 8 --scene c4 variants/*.so 2>&1 | tail -3
