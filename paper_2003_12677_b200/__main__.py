"""python -m paper_2003_12677_b200 recon ... (cli.py)."""
from .cli import main

raise SystemExit(main())
