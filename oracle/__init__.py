"""TEST INFRASTRUCTURE ONLY: CPU checkers (port + compiled reference). See bindings.py."""
