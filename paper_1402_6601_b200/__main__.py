"""``python -m paper_1402_6601_b200 run|sweep|export-dot|validate`` (see cli.py)."""
from .cli import main

raise SystemExit(main())
