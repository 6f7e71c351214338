"""B200-native Mycroft/collsight trace-analysis hot path."""
