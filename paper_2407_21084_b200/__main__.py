"""``python -m paper_2407_21084_b200`` -- the reference CLI's subcommands (cli.py)."""
import sys

from .cli import main

sys.exit(main())
